"""Device-level operations on torch CUDA tensors — one per C-ABI entry point.

PyTorch is only the plumbing here (device memory, the current stream); all
arithmetic runs in libastra_b200.so. Every call is stream-ordered on
torch.cuda.current_stream() and does not synchronise unless stated.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from .errors import ConfigError, NumericalError

REFRESH_FP32_EXACT, REFRESH_BF16, REFRESH_BF16_RERANK, REFRESH_FP8_RERANK = 0, 1, 2, 3
W_FP32, W_BF16 = 0, 1
OPT_SGD, OPT_ADAM = 0, 1
ORIGIN_POS, ORIGIN_HARD, ORIGIN_RAND, ORIGIN_PAD, ORIGIN_IMP = 0, 1, 2, 3, 4
STATUS_NONFINITE_GRAD, STATUS_NONFINITE_GRAD_EMB, STATUS_BOUND_UNSAFE, STATUS_ID_RANGE = 0, 1, 2, 3

_MODES = {"fp32": REFRESH_FP32_EXACT, "fp32_exact": REFRESH_FP32_EXACT, "bf16": REFRESH_BF16,
          "bf16_rerank": REFRESH_BF16_RERANK, "fp8_rerank": REFRESH_FP8_RERANK}


def refresh_mode(mode) -> int:
    if isinstance(mode, int):
        return mode
    try:
        return _MODES[mode]
    except KeyError:
        raise ConfigError(f"unknown refresh mode {mode!r}") from None


class _Workspaces:
    """Per-device scratch buffers grown on demand (one per call site tag)."""

    def __init__(self):
        self._bufs = {}

    def get(self, tag: str, nbytes: int, device) -> torch.Tensor:
        key = (tag, torch.device(device).index)
        buf = self._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
            self._bufs[key] = buf
        return buf


WORKSPACES = _Workspaces()


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _cuda(t, dtype, name):
    if t is None:
        return None
    if not (t.is_cuda and t.dtype == dtype and t.is_contiguous()):
        raise ConfigError(f"{name}: expected a contiguous CUDA {dtype} tensor, got {t.dtype} on {t.device}")
    return t


def f32_to_bf16(x: torch.Tensor) -> torch.Tensor:
    _cuda(x, torch.float32, "f32_to_bf16")
    out = torch.empty(x.shape, dtype=torch.bfloat16, device=x.device)
    _lib.check(_lib.load().astra_f32_to_bf16(_p(x), _p(out), x.numel(), _stream()))
    return out


def quantize_e4m3(x: torch.Tensor) -> torch.Tensor:
    """e4m3 copy (uint8 bytes) of an fp32 / bf16 tensor scaled by 448 / max|x|
    (the FP8_RERANK label snapshot; astra_quantize_e4m3)."""
    if not (x.is_cuda and x.is_contiguous() and x.dtype in (torch.float32, torch.bfloat16)):
        raise ConfigError("quantize_e4m3: expected a contiguous CUDA fp32/bf16 tensor")
    out = torch.empty(x.shape, dtype=torch.uint8, device=x.device)
    scratch = torch.empty(2, dtype=torch.float32, device=x.device)
    _lib.check(_lib.load().astra_quantize_e4m3(_p(x), int(x.dtype == torch.bfloat16), x.numel(), _p(out), _p(scratch),
                                               _stream()))
    return out


def refresh_topk(queries, pos_indptr, pos_ids, k, mode="bf16_rerank", labels_f32=None, labels_bf16=None,
                 label_offset=0, queries_bf16=None, n_labels=None, labels_e4m3=None):
    """Top-k (keys, ids, scores) per query over a label shard, positives
    excluded (retrieve_hard_negatives, anns.py:233-256). keys are int64 views of
    the packed uint64 keys (for astra_topk_merge)."""
    mode = refresh_mode(mode)
    ref = queries if queries is not None else queries_bf16
    nq, d = ref.shape
    if n_labels is None:
        n_labels = next(t for t in (labels_f32, labels_bf16, labels_e4m3) if t is not None).shape[0]
    _cuda(queries, torch.float32, "queries")
    _cuda(labels_f32, torch.float32, "labels_f32")
    _cuda(labels_bf16, torch.bfloat16, "labels_bf16")
    _cuda(queries_bf16, torch.bfloat16, "queries_bf16")
    _cuda(labels_e4m3, torch.uint8, "labels_e4m3")
    _cuda(pos_indptr, torch.int64, "pos_indptr")
    _cuda(pos_ids, torch.int32, "pos_ids")
    lib = _lib.load()
    dev = ref.device
    ws_n = lib.astra_refresh_workspace_size(nq, n_labels, d, k, mode)
    ws = WORKSPACES.get("refresh", ws_n, dev)
    keys = torch.empty((nq, k), dtype=torch.int64, device=dev)
    ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
    scores = torch.empty((nq, k), dtype=torch.float32, device=dev)
    _lib.check(lib.astra_refresh_topk(
        _p(queries), _p(queries_bf16), nq, d, _p(labels_f32), _p(labels_bf16), _p(labels_e4m3), n_labels, label_offset,
        _p(pos_indptr), _p(pos_ids), k, mode, _p(keys), _p(ids), _p(scores), _p(ws), ws.numel(), _stream()))
    return keys, ids, scores


def refresh_plan_j(nq, n_labels, d, k) -> int:
    """j of the label-sharded candidate pass's sample statistics for nq
    queries over n_labels labels and k' = k candidates (0: the shape does not
    run the two-pass plan)."""
    return int(_lib.load().astra_refresh_plan_j(nq, n_labels, d, k))


def refresh_sharded_stage(stage, queries, pos_indptr, pos_ids, k, labels_bf16, label_offset=0, tau_keys=None,
                          io_keys=None, flags=None):
    """One stage of the label-sharded BF16 candidate pass (astra_refresh_sharded_stage):
    1 -> sample_top [nq, j] int32 (orderable score bits of the shard's j largest
         sampled group maxima per query);
    2 -> (keys [nq, k] int64, counts [nq] int32, overflow flags [nq] int32) for
         the global thresholds tau_keys [nq] int64;
    3 -> io_keys rows of the flagged queries (flags [nq] int32) replaced by the
         shard's exact top-k (in place); returns io_keys."""
    _cuda(queries, torch.float32, "queries")
    _cuda(labels_bf16, torch.bfloat16, "labels_bf16")
    _cuda(pos_indptr, torch.int64, "pos_indptr")
    _cuda(pos_ids, torch.int32, "pos_ids")
    nq, d = queries.shape
    L = labels_bf16.shape[0]
    lib = _lib.load()
    mode = refresh_mode("bf16")
    dev = queries.device
    ws = WORKSPACES.get("refresh", lib.astra_refresh_workspace_size(nq, L, d, k, mode), dev)
    top = keys = counts = None
    if stage == 1:
        j = refresh_plan_j(nq, L, d, k)
        if j <= 0:
            raise ConfigError("sharded refresh: this shape does not run the two-pass plan")
        top = torch.empty((nq, j), dtype=torch.int32, device=dev)
    elif stage == 2:
        _cuda(tau_keys, torch.int64, "tau_keys")
        keys = torch.empty((nq, k), dtype=torch.int64, device=dev)
        counts = torch.empty(nq, dtype=torch.int32, device=dev)
        flags = torch.empty(nq, dtype=torch.int32, device=dev)
    else:
        _cuda(flags, torch.int32, "flags")
        _cuda(io_keys, torch.int64, "io_keys")
        keys = io_keys
    _lib.check(lib.astra_refresh_sharded_stage(
        stage, _p(queries), None, nq, d, _p(labels_bf16), L, label_offset, _p(pos_indptr), _p(pos_ids), k, _p(top),
        _p(tau_keys), _p(keys), _p(counts), _p(flags), _p(ws), ws.numel(), _stream()))
    if stage == 1:
        return top
    if stage == 2:
        return keys, counts, flags
    return keys


def rerank_candidates_count(k: int) -> int:
    """k' of the BF16_RERANK candidate pass for a final top-k: max(1.5k, k+16)
    rounded up to 8, <= 2048 (refresh.cu rerank_candidates)."""
    kc = max((3 * k + 1) // 2, k + 16)
    return min((kc + 7) // 8 * 8, 2048)


def rerank_candidates(queries, cand_keys, k, labels_f32=None, labels_bf16=None, label_offset=0):
    """fp32 re-rank of given candidate keys (int64 views; 0 = none) against the
    fp32 (else bf16) label rows: (keys, ids, scores) of the best k per query
    (astra_rerank_candidates)."""
    _cuda(queries, torch.float32, "queries")
    _cuda(cand_keys, torch.int64, "cand_keys")
    _cuda(labels_f32, torch.float32, "labels_f32")
    _cuda(labels_bf16, torch.bfloat16, "labels_bf16")
    labels = labels_f32 if labels_f32 is not None else labels_bf16
    if labels is None:
        raise ConfigError("rerank_candidates: labels_f32 or labels_bf16 required")
    nq, d = queries.shape
    kc = cand_keys.shape[1]
    dev = queries.device
    keys = torch.empty((nq, k), dtype=torch.int64, device=dev)
    ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
    scores = torch.empty((nq, k), dtype=torch.float32, device=dev)
    _lib.check(_lib.load().astra_rerank_candidates(
        _p(queries), nq, d, _p(cand_keys.contiguous()), kc, _p(labels), 0 if labels_f32 is not None else 1,
        label_offset, k, _p(keys), _p(ids), _p(scores), _stream()))
    return keys, ids, scores


def refresh_flagged(nq, n_labels, d, k, mode, device=None) -> int:
    """Queries of the last refresh_topk call of this shape (on this device)
    that the two-pass plan sent to the exact verify pass; -1 when the shape
    runs the single-pass running top-k. Synchronises the current stream."""
    mode = refresh_mode(mode)
    lib = _lib.load()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    ws_n = lib.astra_refresh_workspace_size(nq, n_labels, d, k, mode)
    ws = WORKSPACES.get("refresh", ws_n, dev)
    out = C.c_int64(0)
    _lib.check(lib.astra_refresh_flagged(_p(ws), ws.numel(), nq, n_labels, d, k, mode, C.byref(out), _stream()))
    return int(out.value)


def topk_merge(part_keys: torch.Tensor, k_out: int):
    """Merge [n_parts, nq, k_in] partial key lists into the global top-k_out."""
    _cuda(part_keys, torch.int64, "part_keys")
    n_parts, nq, k_in = part_keys.shape
    lib = _lib.load()
    dev = part_keys.device
    ws = WORKSPACES.get("merge", lib.astra_merge_workspace_size(nq, k_out), dev)
    keys = torch.empty((nq, k_out), dtype=torch.int64, device=dev)
    ids = torch.empty((nq, k_out), dtype=torch.int32, device=dev)
    scores = torch.empty((nq, k_out), dtype=torch.float32, device=dev)
    _lib.check(lib.astra_topk_merge(_p(part_keys), nq, n_parts, k_in, k_out, _p(keys), _p(ids), _p(scores), _p(ws),
                                    ws.numel(), _stream()))
    return keys, ids, scores


def importance_split(ids, scores, k_h):
    """(hard [nq, k_h], cand [nq, n_c], cand_q [nq, n_c]) from a refresh of
    top-(k_h + n_c) per row: H, the importance candidates C and their stored
    draw weights sigmoid(stale score) (astra_importance_split)."""
    _cuda(ids, torch.int32, "ids")
    _cuda(scores, torch.float32, "scores")
    nq, k_tot = ids.shape
    if not 0 <= k_h <= k_tot:
        raise ConfigError(f"importance_split: k_h={k_h} outside [0, {k_tot}]")
    dev = ids.device
    hard = torch.empty((nq, k_h), dtype=torch.int32, device=dev)
    cand = torch.empty((nq, k_tot - k_h), dtype=torch.int32, device=dev)
    cand_q = torch.empty((nq, k_tot - k_h), dtype=torch.float32, device=dev)
    _lib.check(_lib.load().astra_importance_split(_p(ids), _p(scores), nq, k_tot, k_h, _p(hard), _p(cand), _p(cand_q),
                                                  _stream()))
    return hard, cand, cand_q


def sample_slates(seed, epoch, step, rows, pos_indptr, pos_ids, hard, k_h, n_labels, k_p, k_r,
                  cand=None, cand_q=None, k_i=0):
    """Philox negative-mixture slates: (ids int32, y int8, origin int8, weights fp32), B x S."""
    _cuda(rows, torch.int64, "rows")
    _cuda(pos_indptr, torch.int64, "pos_indptr")
    _cuda(pos_ids, torch.int32, "pos_ids")
    B = rows.shape[0]
    dev = rows.device
    if hard is None or k_h == 0:
        hard, k_h, hard_stride = None, 0, 1
    else:
        _cuda(hard, torch.int32, "hard")
        hard_stride = hard.shape[1]
    n_c, cand_stride = 0, 1
    if cand is not None and k_i > 0:
        _cuda(cand, torch.int32, "cand")
        _cuda(cand_q, torch.float32, "cand_q")
        n_c = cand_stride = cand.shape[1]
    else:
        cand = cand_q = None
        k_i = 0
    S = k_p + k_h + k_i + k_r
    ids = torch.empty((B, S), dtype=torch.int32, device=dev)
    y = torch.empty((B, S), dtype=torch.int8, device=dev)
    origin = torch.empty((B, S), dtype=torch.int8, device=dev)
    weights = torch.empty((B, S), dtype=torch.float32, device=dev)
    _lib.check(_lib.load().astra_sample_slates(
        seed & 0xFFFFFFFFFFFFFFFF, epoch & 0xFFFFFFFF, step & 0xFFFFFFFF, _p(rows), B, _p(pos_indptr), _p(pos_ids),
        _p(hard), hard_stride, k_h, _p(cand), _p(cand_q), cand_stride, n_c, k_i, n_labels, k_p, k_r,
        _p(ids), _p(y), _p(origin), _p(weights), _stream()))
    return ids, y, origin, weights


class StepResult:
    """Device outputs of one slate step; `loss`/`status` sync only when read."""

    def __init__(self, loss, grad_emb, status, factors):
        self.loss_dev = loss
        self.grad_emb = grad_emb
        self.status = status
        self.factors = factors

    def status_host(self):
        return self.status.cpu().tolist()

    @property
    def loss(self) -> float:
        return float(self.loss_dev.item())


def slate_step(emb, ids, y, origin, weights, W, lr, weight_decay=0.0, keep=None, factors_in=None,
               optimizer="sgd", adam_m=None, adam_v=None, adam_step=1, betas=(0.9, 0.999), eps=1e-8,
               label_offset=0, want_factors=False, w_absmax=None) -> StepResult:
    """Fused sampled-BCE fwd/bwd + sparse row update of W (trainer.py:366-394).

    origin/weights may be S-vectors (the reference's row-0 semantics) or B x S.
    w_absmax: optional fp32[1] CUDA tensor, a running bound on max|W| kept
    current by the call (enables the single label-major pass)."""
    _cuda(emb, torch.float32, "emb")
    _cuda(keep, torch.float32, "keep")
    _cuda(ids, torch.int32, "ids")
    _cuda(y, torch.int8, "y")
    _cuda(origin, torch.int8, "origin")
    _cuda(weights, torch.float32, "weights")
    _cuda(factors_in, torch.float32, "factors_in")
    _cuda(w_absmax, torch.float32, "w_absmax")
    if W.dtype not in (torch.float32, torch.bfloat16) or not W.is_cuda or not W.is_contiguous():
        raise ConfigError("W must be a contiguous CUDA fp32/bf16 tensor")
    B, S = ids.shape
    d = emb.shape[1]
    Lloc = W.shape[0]
    opt = OPT_ADAM if optimizer == "adam" else OPT_SGD
    if opt == OPT_ADAM:
        _cuda(adam_m, torch.float32, "adam_m")
        _cuda(adam_v, torch.float32, "adam_v")
    o_stride = 0 if origin.dim() == 1 else S
    w_stride = 0 if weights.dim() == 1 else S
    lib = _lib.load()
    dev = emb.device
    ws = WORKSPACES.get("step", lib.astra_step_workspace_size(B, S, d, Lloc), dev)
    grad_emb = torch.empty((B, d), dtype=torch.float32, device=dev)
    loss = torch.empty(1, dtype=torch.float64, device=dev)
    status = torch.empty(4, dtype=torch.int32, device=dev)
    factors = torch.empty((B, S), dtype=torch.float32, device=dev) if want_factors else None
    _lib.check(lib.astra_slate_step(
        _p(emb), _p(keep), _p(ids), _p(y), _p(origin), o_stride, _p(weights), w_stride, _p(factors_in), B, S, d,
        _p(W), W_BF16 if W.dtype == torch.bfloat16 else W_FP32, _p(adam_m), _p(adam_v), opt, Lloc, label_offset,
        float(lr), float(weight_decay), float(betas[0]), float(betas[1]), float(eps), int(adam_step),
        _p(grad_emb), _p(loss), _p(status), _p(factors), _p(w_absmax), _p(ws), ws.numel(), _stream()))
    return StepResult(loss, grad_emb, status, factors)


def dense_bce(scores, pos_indptr, pos_ids, want_grad=True):
    """Elementwise half of the all-negatives arm over B x L scores (fp32, or
    fp64 for the probe): (G = f32(sigmoid) - y or None, float64 loss sum as a
    1-element device tensor). trainer.py:595-597, :401-402."""
    if scores.dtype not in (torch.float32, torch.float64) or not scores.is_cuda or not scores.is_contiguous():
        raise ConfigError("scores must be a contiguous CUDA fp32/fp64 tensor")
    _cuda(pos_indptr, torch.int64, "pos_indptr")
    _cuda(pos_ids, torch.int32, "pos_ids")
    B, L = scores.shape
    lib = _lib.load()
    ws = WORKSPACES.get("dense", lib.astra_dense_workspace_size(B), scores.device)
    G = torch.empty((B, L), dtype=torch.float32, device=scores.device) if want_grad else None
    loss = torch.empty(1, dtype=torch.float64, device=scores.device)
    _lib.check(lib.astra_dense_bce(_p(scores), 1 if scores.dtype == torch.float64 else 0, B, L, _p(pos_indptr),
                                   _p(pos_ids), _p(G), _p(loss), _p(ws), ws.numel(), _stream()))
    return G, loss


def dense_sgd(W, grads, lr, weight_decay=0.0):
    """W -= f32(lr) (grads + f32(wd) W) over every element (trainer.py:604-606)."""
    _cuda(W, torch.float32, "W")
    _cuda(grads, torch.float32, "grads")
    if grads.shape != W.shape:
        raise ConfigError("dense_sgd: grads must have W's shape")
    _lib.check(_lib.load().astra_dense_sgd(_p(W), _p(grads), W.numel(), float(lr), float(weight_decay), _stream()))


def gemm_f32(a, b, a_t=False, b_t=False):
    """D = op(a) op(b)^T in fp32 accuracy on the tf32 tensor cores
    (astra_gemm_f32, 3xTF32). a: [M, K] (a_t: given as [K, M]); b: [N, K]
    (b_t: given as [K, N]). Returns D [M, N] fp32."""
    _cuda(a, torch.float32, "a")
    _cuda(b, torch.float32, "b")
    a, b = a.contiguous(), b.contiguous()
    M, K = (a.shape[1], a.shape[0]) if a_t else (a.shape[0], a.shape[1])
    N, Kb = (b.shape[1], b.shape[0]) if b_t else (b.shape[0], b.shape[1])
    if K != Kb:
        raise ConfigError(f"gemm_f32: inner dimensions differ ({K} vs {Kb})")
    lib = _lib.load()
    ws = WORKSPACES.get("gemm_f32", lib.astra_gemm_f32_workspace_size(M, N, K), a.device)
    D = torch.empty((M, N), dtype=torch.float32, device=a.device)
    _lib.check(lib.astra_gemm_f32(_p(a), 0 if a_t else 1, _p(b), 0 if b_t else 1, M, N, K, _p(D), _p(ws), ws.numel(),
                                  _stream()))
    return D


def full_loss_forward(emb_used, W, pos_indptr, pos_ids, keep=None):
    """One batch of the all-negatives arm before the update (trainer.py:593-599):
    scores = emb_used W^T, G and the float64 loss (astra_dense_bce),
    grad_emb = G W (x keep); both GEMMs astra_gemm_f32 (3xTF32 tensor cores).
    Returns (loss_dev, G, grad_emb)."""
    _cuda(emb_used, torch.float32, "emb_used")
    _cuda(W, torch.float32, "W")
    _cuda(keep, torch.float32, "keep")
    scores = gemm_f32(emb_used, W)
    G, loss = dense_bce(scores, pos_indptr, pos_ids)
    del scores
    grad_emb = gemm_f32(G, W, b_t=True)
    if keep is not None:
        grad_emb = grad_emb * keep
    return loss, G, grad_emb


def full_loss_update(W, G, emb_used, lr, weight_decay=0.0):
    """W -= f32(lr) (G^T emb_used + f32(wd) W) (trainer.py:602-606); the GEMM
    on the tensor cores (astra_gemm_f32)."""
    dense_sgd(W, gemm_f32(G, emb_used, a_t=True, b_t=True), lr, weight_decay)


def dense_probe_loss(emb, W, pos_indptr, pos_ids):
    """float64 dense BCE sum over a probe set (trainer.py:398-403, before the
    division): an fp64 GEMM (cuBLAS DGEMM) and astra_dense_bce in fp64."""
    _cuda(emb, torch.float64, "emb")
    scores = torch.matmul(emb, W.to(torch.float64).t())
    return dense_bce(scores, pos_indptr, pos_ids, want_grad=False)[1]


def raise_for_step_status(status) -> None:
    """Host check of a step's status words (syncs). Mirrors the reference's
    NumericalError raises (classifiers.py:79-80, encoder.py:145-146)."""
    s = status.cpu().tolist() if torch.is_tensor(status) else list(status)
    if s[STATUS_NONFINITE_GRAD_EMB]:
        raise NumericalError("non-finite upstream gradients")
    if s[STATUS_NONFINITE_GRAD]:
        raise NumericalError("non-finite classifier gradient")


def apply_updates(W, ids, grads, lr, weight_decay=0.0):
    """apply_classifier_updates_arrays on device (classifiers.py:75-82); syncs
    to raise NumericalError without writing when a gradient is non-finite."""
    _cuda(ids, torch.int64, "ids")
    _cuda(grads, torch.float32, "grads")
    status = torch.zeros(4, dtype=torch.int32, device=W.device)
    _lib.check(_lib.load().astra_apply_updates(
        _p(W), W_BF16 if W.dtype == torch.bfloat16 else W_FP32, W.shape[0], W.shape[1], _p(ids), _p(grads),
        ids.shape[0], float(lr), float(weight_decay), _p(status), _stream()))
    if status[STATUS_NONFINITE_GRAD].item():
        raise NumericalError("non-finite classifier gradient")
