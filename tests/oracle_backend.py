"""A CPU stand-in for paper_2409_20156_b200.ops built on the ORACLE — test
infrastructure only.

It lets the host-side logic (the reference-facing mirror, install(), the
label-sharded engine and its collectives) run in the build container without
a GPU, e.g. under gloo with world_size 2, or underneath the reference's own
test-suite. It is injected explicitly (install(backend=...) /
ClassifierEngine(backend=...)); the product never selects it.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import torch

from oracle import c_oracle as co
from oracle import xcmix_port as port
from paper_2409_20156_b200.errors import ConfigError, NumericalError
from paper_2409_20156_b200.ops import StepResult, raise_for_step_status  # noqa: F401  (pure host helpers)

DEVICE = "cpu"


def _np(t):
    return None if t is None else t.detach().cpu().numpy()


def f32_to_bf16(x):
    return x.to(torch.bfloat16)


def quantize_e4m3(x):
    return (x.float() * (448.0 / max(float(x.abs().max()), 1e-30))).to(torch.float8_e4m3fn).view(torch.uint8)


def _bf16_f32(x):
    return torch.as_tensor(x).to(torch.bfloat16).float().numpy()


def rerank_candidates_count(k):
    kc = max((3 * k + 1) // 2, k + 16)
    return min((kc + 7) // 8 * 8, 2048)


def _exact_keys(Q, W, label_offset):
    """fp32 FP32_EXACT keys of every (query, label): [nq, L] uint64."""
    nq, L = Q.shape[0], W.shape[0]
    no_pos = np.zeros(nq + 1, np.int64)
    keys, _, _ = co.refresh_fp32(Q, W, no_pos, np.zeros(0, np.int32), L, label_offset)
    ids = co.key_to_id(keys)
    out = np.zeros((nq, L), np.uint64)
    np.put_along_axis(out, (ids - label_offset).astype(np.int64), keys, axis=1)
    return out


def rerank_candidates(queries, cand_keys, k, labels_f32=None, labels_bf16=None, label_offset=0):
    W = _np(labels_f32) if labels_f32 is not None else _np(labels_bf16.float())
    Q = _np(queries)
    ck = _np(cand_keys).view(np.uint64)
    ex = _exact_keys(Q, W, label_offset)
    out = np.zeros((Q.shape[0], k), np.uint64)
    for q in range(Q.shape[0]):
        c = ck[q][ck[q] > 0]
        kk = np.sort(ex[q][(co.key_to_id(c) - label_offset).astype(np.int64)])[::-1][:k]
        out[q, : len(kk)] = kk
    ids = np.where(out > 0, co.key_to_id(out), -1).astype(np.int32)
    scores = np.where(out > 0, co.key_to_score(out), -np.inf).astype(np.float32)
    return torch.from_numpy(out.view(np.int64)), torch.from_numpy(ids), torch.from_numpy(scores)


# The label-sharded candidate pass (stand-ins with the GPU stages' contract:
# the sample statistics are the maxima of 64-label groups of every 2nd
# 256-label tile of the shard, j = 3; candidates are the non-positive labels at
# or above the given threshold; the verify pass is the exact local top-k).
_SHARD_J = 3


def refresh_plan_j(nq, n_labels, d, k):
    return _SHARD_J


def _bf16_keys(queries, labels_bf16, pos_indptr, pos_ids, label_offset, exclude_pos):
    """[nq, L] uint64 keys of the bf16-operand scores (0 for excluded positives)."""
    Q = _bf16_f32(queries)
    W = _np(labels_bf16.float())
    nq, L = Q.shape[0], W.shape[0]
    keys = _exact_keys(Q, W, label_offset)
    if exclude_pos:
        ip, pid = _np(pos_indptr), _np(pos_ids)
        for q in range(nq):
            loc = pid[ip[q]:ip[q + 1]].astype(np.int64) - label_offset
            loc = loc[(loc >= 0) & (loc < L)]
            keys[q, loc] = 0
    return keys


def refresh_sharded_stage(stage, queries, pos_indptr, pos_ids, k, labels_bf16, label_offset=0, tau_keys=None,
                          io_keys=None, flags=None):
    L = labels_bf16.shape[0]
    if stage == 1:
        keys = _bf16_keys(queries, labels_bf16, pos_indptr, pos_ids, label_offset, False)
        ords = (keys >> np.uint64(32)).astype(np.uint32)
        gm = []
        for t0 in range(0, L, 512):  # every 2nd 256-label tile
            for g0 in range(t0, min(t0 + 256, L), 64):
                gm.append(ords[:, g0:min(g0 + 64, L)].max(axis=1))
        gm = np.stack(gm, axis=1)
        top = -np.sort(-gm.astype(np.int64), axis=1)[:, :_SHARD_J]
        if top.shape[1] < _SHARD_J:
            top = np.pad(top, ((0, 0), (0, _SHARD_J - top.shape[1])))
        return torch.from_numpy(top.astype(np.uint32).view(np.int32))
    keys = _bf16_keys(queries, labels_bf16, pos_indptr, pos_ids, label_offset, True)
    nq = keys.shape[0]
    if stage == 2:
        tau = _np(tau_keys).view(np.uint64)
        out = np.zeros((nq, k), np.uint64)
        counts = np.zeros(nq, np.int32)
        for q in range(nq):
            c = keys[q][keys[q] >= max(tau[q], np.uint64(1))]
            c = np.sort(c)[::-1][:k]
            out[q, : len(c)] = c
            counts[q] = len(c)
        return torch.from_numpy(out.view(np.int64)), torch.from_numpy(counts), torch.zeros(nq, dtype=torch.int32)
    out = _np(io_keys).view(np.uint64).copy()
    fl = _np(flags)
    for q in range(nq):
        if fl[q]:
            c = np.sort(keys[q][keys[q] > 0])[::-1][:k]
            out[q] = 0
            out[q, : len(c)] = c
    io_keys.copy_(torch.from_numpy(out.view(np.int64)))
    return io_keys


def refresh_topk(queries, pos_indptr, pos_ids, k, mode="fp32", labels_f32=None, labels_bf16=None, label_offset=0,
                 queries_bf16=None, n_labels=None, labels_e4m3=None):
    """fp32: the C oracle. bf16 / bf16_rerank (stand-ins with the GPU modes'
    structure, for the multi-process protocol tests): the candidate pass ranks
    by the fixed-order fp32 score of bf16-rounded operands; bf16_rerank
    re-scores its top-k' in fp32."""
    if k < 1:
        raise ConfigError("refresh: k must be >= 1")
    if mode in ("bf16", "bf16_rerank"):
        W = _np(labels_bf16.float()) if labels_bf16 is not None else _bf16_f32(labels_f32)
        kc = k if mode == "bf16" else rerank_candidates_count(k)
        keys, ids, scores = co.refresh_fp32(_bf16_f32(queries), W, _np(pos_indptr), _np(pos_ids), kc, label_offset)
        if mode == "bf16":
            return (torch.from_numpy(keys.view(np.int64)), torch.from_numpy(ids), torch.from_numpy(scores))
        return rerank_candidates(queries, torch.from_numpy(keys.view(np.int64)), k, labels_f32=labels_f32,
                                 labels_bf16=labels_bf16, label_offset=label_offset)
    keys, ids, scores = co.refresh_fp32(_np(queries), _np(labels_f32), _np(pos_indptr), _np(pos_ids), k, label_offset)
    return (torch.from_numpy(keys.view(np.int64)), torch.from_numpy(ids), torch.from_numpy(scores))


def topk_merge(part_keys, k_out):
    pk = _np(part_keys).view(np.uint64)
    n_parts, nq, k_in = pk.shape
    allk = np.sort(pk.transpose(1, 0, 2).reshape(nq, n_parts * k_in), axis=1)[:, ::-1][:, :k_out]
    allk = np.ascontiguousarray(allk)
    ids = np.where(allk > 0, co.key_to_id(allk), -1).astype(np.int32)
    scores = np.where(allk > 0, co.key_to_score(allk), -np.inf).astype(np.float32)
    return torch.from_numpy(allk.view(np.int64)), torch.from_numpy(ids), torch.from_numpy(scores)


def sample_slates(seed, epoch, step, rows, pos_indptr, pos_ids, hard, k_h, n_labels, k_p, k_r, cand=None,
                  cand_q=None, k_i=0):
    try:
        out = co.sample_slates(seed, epoch, step, _np(rows), _np(pos_indptr), _np(pos_ids), _np(hard), k_h, n_labels,
                               k_p, k_r, cand=_np(cand), cand_q=_np(cand_q), k_i=k_i)
    except ValueError as e:
        raise ConfigError(str(e)) from None
    return tuple(torch.from_numpy(a) for a in out)


def slate_step(emb, ids, y, origin, weights, W, lr, weight_decay=0.0, keep=None, factors_in=None, optimizer="sgd",
               adam_m=None, adam_v=None, adam_step=1, betas=(0.9, 0.999), eps=1e-8, label_offset=0,
               want_factors=False, w_absmax=None):
    """The reference arithmetic (oracle/xcmix_port.py) restricted to this
    shard's label range [label_offset, label_offset + W.shape[0])."""
    if optimizer != "sgd":
        raise ConfigError("oracle backend: SGD only")
    E = _np(emb)
    I = _np(ids).astype(np.int64)
    Y = _np(y)
    O = _np(origin)
    Wt = _np(W).astype(np.float32, copy=False)
    Wn = W.detach().numpy()  # in-place view
    L_loc = Wn.shape[0]
    B, S = I.shape
    own = (I >= label_offset) & (I < label_offset + L_loc)
    loc = np.where(own, I - label_offset, 0)
    rows_w = Wt[loc]
    if factors_in is None:
        scores = np.einsum("bsd,bd->bs", rows_w, E)
        terms_ok = own
        O2 = O if O.ndim == 2 else np.broadcast_to(O, (B, S))
        W2 = _np(weights) if _np(weights).ndim == 2 else np.broadcast_to(_np(weights), (B, S))
        _, factors = port.slate_factors(scores, Y, O2, W2)
        pos_slot = O2 == port.ORIGIN_POS
        yf = Y.astype(np.float32)
        sp_neg = port.softplus64(-scores)
        lt = (yf * pos_slot) * sp_neg + (W2 * ((1.0 - yf) * (~pos_slot))) * (sp_neg + scores)
        loss = float(lt[terms_ok].sum())
    else:
        factors = _np(factors_in)
        loss = float("nan")
    factors = np.where(own, factors, np.float32(0)).astype(np.float32)
    grad_emb = np.einsum("bs,bsd->bd", factors, rows_w * own[:, :, None])
    if keep is not None:
        grad_emb = grad_emb * _np(keep)
    status = np.zeros(4, np.int32)
    if not np.isfinite(grad_emb).all():
        status[1] = 1
    owned_flat = own.ravel()
    A = sp.csr_matrix((factors.ravel()[owned_flat], loc.ravel()[owned_flat],
                       np.concatenate([[0], np.cumsum(own.sum(axis=1))])), shape=(B, L_loc))
    full = A.T @ E
    uids = np.unique(loc.ravel()[owned_flat])
    grads = np.asarray(full[uids], dtype=np.float32)
    if not np.isfinite(grads).all():
        status[0] = 1
    if not status.any() and len(uids):
        rows = Wn[uids]
        Wn[uids] = rows - np.float32(lr) * (grads + np.float32(weight_decay) * rows)
    return StepResult(torch.tensor([loss], dtype=torch.float64), torch.from_numpy(np.ascontiguousarray(grad_emb, np.float32)),
                      torch.from_numpy(status), torch.from_numpy(factors) if want_factors else None)


def apply_updates(W, ids, grads, lr, weight_decay=0.0):
    Wn = W.detach().numpy()
    try:
        port.apply_classifier_updates_arrays(Wn, _np(ids), _np(grads), lr, weight_decay)
    except port.OracleNumericalError as e:
        raise NumericalError(str(e)) from None


def _dense_y_from_csr(pos_indptr, pos_ids, B, L):
    ip, ids = _np(pos_indptr), _np(pos_ids)
    return port.dense_y([ids[ip[b]:ip[b + 1]] for b in range(B)], L)


def full_loss_forward(emb_used, W, pos_indptr, pos_ids, keep=None):
    e = _np(emb_used)
    yb = _dense_y_from_csr(pos_indptr, pos_ids, e.shape[0], W.shape[0])
    loss, G, grad_emb = port.full_loss_forward(_np(W), e, _np(keep), yb)
    return torch.tensor([loss], dtype=torch.float64), torch.from_numpy(G), torch.from_numpy(grad_emb)


def full_loss_update(W, G, emb_used, lr, weight_decay=0.0):
    port.full_loss_update(W.numpy(), _np(G), _np(emb_used), lr, weight_decay)  # in place (shared memory)


def dense_probe_loss(emb, W, pos_indptr, pos_ids):
    e = _np(emb)
    mask = _dense_y_from_csr(pos_indptr, pos_ids, e.shape[0], W.shape[0]).astype(bool)
    return torch.tensor([port.probe_full_loss(e, _np(W), mask)], dtype=torch.float64)


def importance_split(ids, scores, k_h):
    i, sc = _np(ids), _np(scores).astype(np.float32)
    q = np.where(i[:, k_h:] >= 0, (np.float32(1.0) / (np.float32(1.0) + np.exp(-sc[:, k_h:]))), 0.0).astype(np.float32)
    return (torch.from_numpy(np.ascontiguousarray(i[:, :k_h])), torch.from_numpy(np.ascontiguousarray(i[:, k_h:])),
            torch.from_numpy(q))
