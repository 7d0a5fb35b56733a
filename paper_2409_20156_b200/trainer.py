"""Drop-in for the classifier half of xcmix.trainer's hot loop.

  _assemble_batch_slates(state, batch_rows, epoch, rng, hard_batch)
        -> (ids B x S int64, y B x S int8, origin S int8, weights S fp32)   trainer.py:262-318
  _batch_forward_backward(state, batch_rows, epoch, rng, step_lr_enc,
                          step_lr_clf, feats=None) -> float               trainer.py:336-395
  _probe_full_loss(state) -> float                                        trainer.py:398-403
  _eval_p_at(state) -> (p@1, p@5)                                         trainer.py:406-423
  train_full_loss_baseline(dataset, config, eval_dataset=None,
                           checkpoint_path=None)                          trainer.py:563-616

Slates come from the Philox sampler (astra_sample_slates) keyed by one 63-bit
draw from the caller's generator, so runs stay bitwise reproducible and the
generator advances deterministically; origin/weights are returned the way the
reference does (row 0's origin vector, trainer.py:313). The classifier step
(gather, loss, factors, grad_emb, per-label sums, SGD update) runs in
astra_slate_step on a device-resident copy of bank.weights (bank.DeviceBank):
the device copy is authoritative while training and host reads of
bank.weights (refresh snapshot, checkpoint, evaluation) copy it back lazily.
The encoder (embed_batch / encoder_backward_batch / adam_step) stays the
caller's (the reference's) — it is outside the hot path.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _backend
from .bank import DeviceBank, device_weights
from .errors import ConfigError, NumericalError

# The drop-in's classifier step is bitwise run-to-run reproducible by default
# (the reference's determinism contract, test_acceptance.py:462-474): the
# two-kernel schedule sums grad_emb in a fixed order. FAST_STEP = True (or
# install(fast_step=True) / ASTRA_DROPIN_FAST_STEP=1) takes the single
# label-major pass instead (same W', grad_emb summed in arrival order).
FAST_STEP = os.environ.get("ASTRA_DROPIN_FAST_STEP") == "1"



def curriculum_counts(epoch: int, strategy, tau_s: int) -> tuple[int, int]:
    """Effective (hard, random) slot counts: the caller's own
    xcmix.sampler.curriculum_counts (sampler.py:82-94), not a restatement."""
    from xcmix.sampler import curriculum_counts as reference_counts

    return reference_counts(epoch, strategy, tau_s)


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
    ids, y, origin, weights = _slates_device(state, batch_rows, epoch, rng, hard_batch)
    return (ids.cpu().numpy().astype(np.int64), y.cpu().numpy(), origin[0].cpu().numpy(),
            weights[0].cpu().numpy())


def _slates_device(state, batch_rows, epoch, rng, hard_batch):
    """The slates of _assemble_batch_slates as device tensors (ids [B, S]
    int32, y [B, S] int8, origin / weights [B, S]); consumes the caller's
    generator exactly as _assemble_batch_slates does (one 63-bit draw)."""
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
    return ops.sample_slates(seed, int(epoch), 0, torch.from_numpy(rows).to(dev), torch.from_numpy(indptr).to(dev),
                             torch.from_numpy(pos).to(dev), hard, k_h_eff, L, cfg.k_p, k_r_eff)


def _uptodate_hard_batch(state, batch_rows, embeddings, epoch):
    """UpToDateHard (trainer.py:321-333): per row, the top k_h_eff labels of
    the CURRENT classifier by exact inner product, positives dropped, ties to
    the lower id. The reference builds a fresh exact index from a host copy
    of W and runs one query per row; here it is one batched fp32-exact MIPS
    launch over the batch against the live device weights (no snapshot, no
    upload). Counters follow the reference (index_queries += rows); no
    host-side live_index is built."""
    k_h_eff, _ = curriculum_counts(epoch, state.strategy, state.config.tau_s)
    rows = np.asarray(batch_rows, dtype=np.int64)
    out = np.empty((len(rows), k_h_eff), dtype=np.int64)
    if k_h_eff == 0 or len(rows) == 0:
        return out
    positives = [state.dataset.positives[i] for i in rows]
    W = DeviceBank.attach(state.bank).W
    if k_h_eff + max(len(p) for p in positives) > W.shape[0]:
        raise ConfigError("k_h plus the positive count exceeds the label count")
    state.caches.index_queries += len(rows)
    indptr, ids = _csr(positives)
    dev = W.device
    ops = _backend.get()
    _, top, _ = ops.refresh_topk(torch.from_numpy(np.ascontiguousarray(embeddings, dtype=np.float32)).to(dev),
                                 torch.from_numpy(indptr).to(dev), torch.from_numpy(ids).to(dev), k_h_eff, "fp32",
                                 labels_f32=W)
    out[:] = top.cpu().numpy()
    return out


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

    ops = _backend.get()
    dev = _backend.device()
    if xt._assemble_batch_slates is _assemble_batch_slates:
        # the installed sampler: its slates stay on the device (no host round trip)
        ids_d, y_d, origin_d, weights_d = _slates_device(state, batch_rows, epoch, rng, hard_batch)
        origin_d, weights_d = origin_d[0], weights_d[0]
    else:  # a caller-provided slate function (e.g. the reference's, ASTRA_DROPIN_SLATES=reference)
        ids, y, origin, weights = xt._assemble_batch_slates(state, batch_rows, epoch, rng, hard_batch)
        ids_d = torch.from_numpy(np.ascontiguousarray(ids, dtype=np.int32)).to(dev)
        y_d = torch.from_numpy(np.ascontiguousarray(y, dtype=np.int8)).to(dev)
        origin_d = torch.from_numpy(np.ascontiguousarray(origin, dtype=np.int8)).to(dev)
        weights_d = torch.from_numpy(np.ascontiguousarray(weights, dtype=np.float32)).to(dev)
    bank = DeviceBank.attach(state.bank)
    res = ops.slate_step(
        torch.from_numpy(np.ascontiguousarray(emb_used, dtype=np.float32)).to(dev), ids_d, y_d,
        origin_d.contiguous(), weights_d.contiguous(), bank.W, float(step_lr_clf),
        float(cfg.weight_decay_classifier),
        keep=None if keep is None else torch.from_numpy(np.ascontiguousarray(keep)).to(dev),
        w_absmax=bank.w_absmax if FAST_STEP else None)
    grad_emb = res.grad_emb.cpu().numpy()
    status = res.status_host()
    # encoder half stays with the caller; it raises NumericalError on a
    # non-finite grad_emb before updating anything (encoder.py:145-146)
    enc_grads = xt.encoder_backward_batch(state.encoder, feats, grad_emb)
    xt.adam_step(state.opt, state.encoder, enc_grads, step_lr_enc)
    if status[1] or status[0]:
        raise NumericalError("non-finite classifier gradient")  # classifiers.py:79-80; W untouched
    bank.mark_updated()
    return res.loss


# ------------------------------------------------------------ dense arms


def _csr(rows_positives):
    """CSR (indptr int64, sorted distinct ids int32) of per-row positive lists."""
    from .anns import positives_csr

    return positives_csr(list(rows_positives), unique=True)


def _dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a if dtype is None else np.asarray(a, dtype=dtype)))
    return t.to(_backend.device())


def _host_weights(state):
    """The bank's current weights on the device (the live device copy when
    the drop-in trains this bank, else an upload of the host array)."""
    return device_weights(state.bank)


def _probe_full_loss(state) -> float:
    """Dense float64 BCE over the probe rows (trainer.py:398-403): fp64 cuBLAS
    GEMM + astra_dense_bce instead of the 200 x L host computation."""
    import xcmix.trainer as xt

    emb = xt.embed_batch(state.encoder, state.probe_feats).astype(np.float64)
    pos = np.asarray(state.probe_y, dtype=bool)
    indptr, ids = _csr([np.nonzero(r)[0] for r in pos])
    ops = _backend.get()
    total = ops.dense_probe_loss(_dev(emb), _host_weights(state), _dev(indptr), _dev(ids))
    return float(float(total.item()) / len(state.probe_rows))


def _eval_p_at(state):
    """P@1 / P@5 on the eval set (trainer.py:406-423): the top-5 of every
    point by the exact fp32 MIPS kernel (descending score, ties -> lower id,
    = the reference's stable argsort) instead of a dense host argsort."""
    import xcmix.trainer as xt

    ds = state.eval_dataset
    if ds is None:
        return None, None
    emb = xt.embed_batch(state.encoder, ds.features)
    L = state.bank.weights.shape[0]
    k = min(5, L)
    n_pts = emb.shape[0]
    ops = _backend.get()
    no_pos = _dev(np.zeros(n_pts + 1, dtype=np.int64))
    _, top, _ = ops.refresh_topk(_dev(emb, np.float32), no_pos, _dev(np.zeros(0, np.int32)), k, "fp32",
                                 labels_f32=_host_weights(state))
    top5 = top.cpu().numpy()
    hits1 = hits5 = n = 0
    for i in range(ds.n_points):
        pos = set(ds.positives[i].tolist())
        if not pos:
            continue
        n += 1
        hits1 += int(top5[i, 0] in pos)
        hits5 += len(pos.intersection(top5[i].tolist())) / 5.0
    if n == 0:
        return None, None
    return hits1 / n, hits5 / n


def train_full_loss_baseline(dataset, config, eval_dataset=None, checkpoint_path=None):
    """All-negatives arm (trainer.py:563-616) with the classifier on the GPU:
    per batch, scores / G / loss / grad_emb (fp32 cuBLAS GEMMs +
    astra_dense_bce), then the caller's encoder backward + Adam, then the dense
    SGD of every row (astra_dense_sgd). The generator stream, batch order,
    dropout and the encoder path are the reference's; bank.weights is written
    back after every epoch (before the epoch's probe / eval)."""
    import time

    import xcmix.trainer as xt

    if dataset.n_labels > xt._FULL_LOSS_LABEL_CAP:
        raise ConfigError(f"full-loss baseline capped at L <= {xt._FULL_LOSS_LABEL_CAP}")
    state = xt.TrainerState(dataset, config, eval_dataset)
    n_batches = -(-len(state.active_rows) // config.batch_size)
    state.total_steps = max(config.epochs * n_batches, 1)
    ops = _backend.get()
    mirror = DeviceBank.attach(state.bank)
    W = mirror.W
    for epoch in range(config.epochs):
        t0 = time.perf_counter()
        rng = np.random.default_rng((config.seed, 7919, epoch))
        perm = rng.permutation(len(state.active_rows))
        rows = state.active_rows[perm]
        total_loss = 0.0
        for start in range(0, len(rows), config.batch_size):
            batch = rows[start : start + config.batch_size]
            lr_enc = xt.lr_at(state.global_step, state.total_steps, config.warmup_steps, config.lr_encoder)
            lr_clf = xt.lr_at(state.global_step, state.total_steps, config.warmup_steps, config.lr_classifier)
            feats = dataset.features[batch]
            emb = xt.embed_batch(state.encoder, feats)
            if config.dropout > 0:
                keep = (rng.random(emb.shape) >= config.dropout).astype(np.float32) / np.float32(1.0 - config.dropout)
                emb_used = emb * keep
            else:
                keep = None
                emb_used = emb
            indptr, ids = _csr([dataset.positives[r] for r in batch])
            emb_d = _dev(emb_used, np.float32)
            loss, G, grad_emb = ops.full_loss_forward(emb_d, W, _dev(indptr), _dev(ids),
                                                      keep=None if keep is None else _dev(keep))
            total_loss += float(loss.item())
            enc_grads = xt.encoder_backward_batch(state.encoder, feats, grad_emb.cpu().numpy())
            xt.adam_step(state.opt, state.encoder, enc_grads, lr_enc)
            ops.full_loss_update(W, G, emb_d, lr_clf, config.weight_decay_classifier)
            mirror.mark_updated()
            state.global_step += 1
        wall = time.perf_counter() - t0
        evaluate_now = (epoch % config.eval_every == config.eval_every - 1) or epoch == config.epochs - 1
        p1, p5 = xt._eval_p_at(state) if evaluate_now else (None, None)
        state.log.records.append(
            xt.EpochRecord(epoch, wall, total_loss / max(len(rows), 1), xt._probe_full_loss(state), p1, p5, -1)
        )
    if checkpoint_path is not None:
        xt.save_checkpoint(checkpoint_path, state.encoder, state.bank, config)
    return state.encoder, state.bank, state.log
