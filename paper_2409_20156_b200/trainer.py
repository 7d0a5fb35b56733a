"""Drop-in for the classifier half of xcmix.trainer's hot loop.

  _assemble_batch_slates(state, batch_rows, epoch, rng, hard_batch)
        -> (ids B x S int64, y B x S int8, origin S int8, weights S fp32)   trainer.py:262-318
  _batch_forward_backward(state, batch_rows, epoch, rng, step_lr_enc,
                          step_lr_clf, feats=None) -> float               trainer.py:336-395

Slates come from the Philox sampler (astra_sample_slates) keyed by one 63-bit
draw from the caller's generator, so runs stay bitwise reproducible and the
generator advances deterministically; origin/weights are returned the way the
reference does (row 0's origin vector, trainer.py:313). The classifier step
(gather, loss, factors, grad_emb, per-label sums, SGD update) runs in
astra_slate_step on a device mirror of bank.weights; touched rows are written
back so bank.weights stays the authoritative host copy for eval/checkpoints.
The encoder (embed_batch / encoder_backward_batch / adam_step) stays the
caller's (the reference's) — it is outside the hot path.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _backend
from .errors import ConfigError, NumericalError

_HARD_ONLY = {"StaleHard", "UpToDateHard", "LabelEmbHard"}
_MIXTURES = {"Mixture", "LabelEmbMixture"}


def curriculum_counts(epoch: int, strategy, tau_s: int) -> tuple[int, int]:
    """Effective (hard, random) slot counts, restating sampler.py:82-94."""
    total = strategy.k_h + strategy.k_r
    if epoch < tau_s or strategy.kind == "RandomOnly":
        return 0, total
    if strategy.kind in _HARD_ONLY:
        return total, 0
    if strategy.kind in _MIXTURES:
        return strategy.k_h, strategy.k_r
    frac = min(1.0, (epoch - tau_s) / strategy.curriculum_ramp)
    k_h_eff = int(round(strategy.k_h * frac))
    return k_h_eff, total - k_h_eff


class DeviceBank:
    """Device mirror of a ClassifierBank's fp32 weights (created on first use,
    rebuilt if bank.weights is replaced by another array object)."""

    def __init__(self, host: np.ndarray):
        self.host = host
        self.W = torch.from_numpy(np.ascontiguousarray(host, dtype=np.float32)).to(_backend.device())

    @classmethod
    def for_bank(cls, owner, bank) -> "DeviceBank":
        db = getattr(owner, "_astra_bank", None)
        if db is None or db.host is not bank.weights:
            db = cls(bank.weights)
            owner._astra_bank = db
        return db

    def sync_rows(self, ids: torch.Tensor) -> None:
        """Copy the given (device) rows back into the host array."""
        idx = ids.to(torch.int64)
        self.host[idx.cpu().numpy()] = self.W[idx].cpu().numpy()


def _positives_csr(state, batch_rows):
    ppad = state.pos_padded[batch_rows]
    npos = state.n_pos[batch_rows]
    indptr = np.zeros(len(batch_rows) + 1, dtype=np.int64)
    np.cumsum(npos, out=indptr[1:])
    ids = np.sort(np.where(ppad >= 0, ppad, np.iinfo(np.int64).max), axis=1)
    flat = ids[np.arange(ppad.shape[1])[None, :] < npos[:, None]].astype(np.int32)
    return indptr, flat


def _assemble_batch_slates(state, batch_rows, epoch, rng, hard_batch):
    """Philox slates for one batch (trainer.py:262-318 contract)."""
    cfg = state.config
    L = state.dataset.n_labels
    k_h_eff = 0 if hard_batch is None else hard_batch.shape[1]
    _, k_r_eff = curriculum_counts(epoch, state.strategy, cfg.tau_s)
    if hard_batch is None:
        k_r_eff = state.strategy.k_h + state.strategy.k_r
    if k_h_eff + 1 > L:
        raise ConfigError("hard set covers the whole label space")
    seed = int(rng.integers(0, 2**63 - 1))
    ops = _backend.get()
    dev = _backend.device()
    rows = np.asarray(batch_rows, dtype=np.int64)
    indptr, pos = _positives_csr(state, rows)
    hard = None if hard_batch is None else torch.from_numpy(np.ascontiguousarray(hard_batch, dtype=np.int32)).to(dev)
    ids, y, origin, weights = ops.sample_slates(
        seed, int(epoch), 0, torch.from_numpy(rows).to(dev), torch.from_numpy(indptr).to(dev),
        torch.from_numpy(pos).to(dev), hard, k_h_eff, L, cfg.k_p, k_r_eff)
    return (ids.cpu().numpy().astype(np.int64), y.cpu().numpy(), origin[0].cpu().numpy(),
            weights[0].cpu().numpy())


def _batch_forward_backward(state, batch_rows, epoch, rng, step_lr_enc, step_lr_clf, feats=None):
    """One mini-batch update; returns the summed slate loss (trainer.py:336-395)."""
    import xcmix.trainer as xt  # the caller's module: encoder, slates, UpToDate arm

    cfg = state.config
    if feats is None:
        feats = state.dataset.features[batch_rows]
    emb = xt.embed_batch(state.encoder, feats)
    if cfg.dropout > 0:
        keep = (rng.random(emb.shape) >= cfg.dropout).astype(np.float32) / np.float32(1.0 - cfg.dropout)
        emb_used = emb * keep
    else:
        keep = None
        emb_used = emb

    use_hard = state.strategy.uses_hard_negatives and epoch >= cfg.tau_s
    hard_batch = None
    if use_hard:
        if state.strategy.kind == "UpToDateHard":
            hard_batch = xt._uptodate_hard_batch(state, batch_rows, emb_used, epoch)
        else:
            if state.caches.negative_cache is None:
                raise ConfigError("hard-negative epoch reached without a cache")
            k_h_eff, _ = curriculum_counts(epoch, state.strategy, cfg.tau_s)
            state.caches.cache_reads += len(batch_rows)
            hard_batch = state.caches.negative_cache.ids[batch_rows][:, :k_h_eff].astype(np.int64)
            if hard_batch.shape[1] == 0:
                hard_batch = None

    ids, y, origin, weights = xt._assemble_batch_slates(state, batch_rows, epoch, rng, hard_batch)

    ops = _backend.get()
    dev = _backend.device()
    bank = DeviceBank.for_bank(state, state.bank)
    ids_d = torch.from_numpy(np.ascontiguousarray(ids, dtype=np.int32)).to(dev)
    res = ops.slate_step(
        torch.from_numpy(np.ascontiguousarray(emb_used, dtype=np.float32)).to(dev), ids_d,
        torch.from_numpy(np.ascontiguousarray(y, dtype=np.int8)).to(dev),
        torch.from_numpy(np.ascontiguousarray(origin, dtype=np.int8)).to(dev),
        torch.from_numpy(np.ascontiguousarray(weights, dtype=np.float32)).to(dev), bank.W, float(step_lr_clf),
        float(cfg.weight_decay_classifier),
        keep=None if keep is None else torch.from_numpy(np.ascontiguousarray(keep)).to(dev))
    grad_emb = res.grad_emb.cpu().numpy()
    status = res.status_host()
    # encoder half stays with the caller; it raises NumericalError on a
    # non-finite grad_emb before updating anything (encoder.py:145-146)
    enc_grads = xt.encoder_backward_batch(state.encoder, feats, grad_emb)
    xt.adam_step(state.opt, state.encoder, enc_grads, step_lr_enc)
    if status[1] or status[0]:
        raise NumericalError("non-finite classifier gradient")  # classifiers.py:79-80; W untouched
    bank.sync_rows(torch.unique(ids_d))
    return res.loss
