"""Drop-in for the exact shortlist refresh of xcmix.anns.

Same names, signatures, return types and error classes as the reference:
  build_exact(vectors, snapshot_epoch=0) -> AnnsIndex            anns.py:99-100
  retrieve_hard_negatives(index, embeddings, positives, k_h,
                          query_beam=128) -> NegativeCache        anns.py:233-268
  query_topk(index, query, k, query_beam=128) -> ScoredLabels     anns.py:211-230
plus query_topk_batch(index, queries, k) -> (ids, scores), the batched form
the exact MIPS kernel is built for (evaluation / UpToDateHard).
The exact branch (anns.py:252-256: E @ W^T, positive mask, _batched_topk) runs
on the GPU (libastra_b200: tcgen05 GEMM + fused top-k, or the fp32-exact SIMT
kernel). The approximate graph index (anns.py:136-208) is outside the B200
path: retrieve_hard_negatives raises ConfigError for it unless install()
recorded the reference implementation to hand it back to.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _backend
from .errors import ConfigError, NumericalError

try:  # reuse the caller's types when running under the reference package
    from xcmix.anns import AnnsIndex, NegativeCache
except ImportError:

    @dataclass
    class AnnsIndex:
        kind: str
        vectors: np.ndarray
        snapshot_epoch: int = 0
        graph: list | None = None
        entry_point: int = 0

        @property
        def size(self) -> int:
            return self.vectors.shape[0]

    @dataclass
    class NegativeCache:
        ids: np.ndarray
        built_from_epoch: int

        @property
        def n_queries(self) -> int:
            return self.ids.shape[0]

        @property
        def k_h(self) -> int:
            return self.ids.shape[1]


try:
    from xcmix.classifiers import ScoredLabels
except ImportError:

    @dataclass
    class ScoredLabels:
        label_ids: np.ndarray
        scores: np.ndarray


# set by install(): the reference implementations for non-exact indexes
_approx_impl = None
_approx_query_impl = None
QUERY_CHUNK = 1 << 16


def _check_vectors(vectors) -> np.ndarray:
    """Contiguous fp32 copy, nonempty 2-D, finite (anns.py:90-96)."""
    vectors = np.ascontiguousarray(vectors, dtype=np.float32)
    if vectors.ndim != 2 or vectors.shape[0] < 1:
        raise ConfigError("index needs a nonempty M x d matrix")
    if not np.isfinite(vectors).all():
        raise NumericalError("non-finite vectors in index build")
    return vectors.copy()


def build_exact(vectors, snapshot_epoch: int = 0) -> AnnsIndex:
    return AnnsIndex(kind="exact", vectors=_check_vectors(vectors), snapshot_epoch=snapshot_epoch)


def refresh_mode_for(d: int, n_labels: int) -> str:
    """fp32-exact unless the tensor-core path applies (ASTRA_REFRESH_MODE overrides)."""
    mode = os.environ.get("ASTRA_REFRESH_MODE", "auto")
    if mode != "auto":
        return mode
    return "bf16_rerank" if d % 64 == 0 and n_labels >= 4096 else "fp32"


def _device_snapshot(index: AnnsIndex, mode: str):
    """Device copies of the immutable index (build_exact copies and freezes its
    vectors, anns.py:90-100), cached on the index: fp32, plus the bf16 or e4m3
    copy the tensor-core candidate pass reads. Returns the refresh_topk label
    keyword arguments for `mode`."""
    ops = _backend.get()
    dev = _backend.device()
    snap = getattr(index, "_astra_snapshot", None)
    if snap is None or snap["vectors"] is not index.vectors or snap["dev"] != dev:
        w32 = torch.from_numpy(np.ascontiguousarray(index.vectors, dtype=np.float32)).to(dev)
        snap = {"vectors": index.vectors, "dev": dev, "f32": w32}
        index._astra_snapshot = snap
    labels = {"labels_f32": snap["f32"]}
    if mode in ("bf16", "bf16_rerank"):
        if "bf16" not in snap:
            snap["bf16"] = ops.f32_to_bf16(snap["f32"])
        labels["labels_bf16"] = snap["bf16"]
    elif mode == "fp8_rerank":
        if "e4m3" not in snap:
            snap["e4m3"] = ops.quantize_e4m3(snap["f32"])
        labels["labels_e4m3"] = snap["e4m3"]
    return labels


def positives_csr(positives, rows=None, unique=False):
    """(indptr int64, ids int32) of per-query positive id arrays, sorted per row
    (and deduplicated per row with unique=True). Vectorised: one concatenate,
    a segmented sort only when some row is out of order (a per-row np.sort /
    np.unique cost ~10 ms per 1024 rows on the host)."""
    if rows is not None:
        positives = [positives[i] for i in rows]
    n = len(positives)
    lens = np.fromiter((len(p) for p in positives), dtype=np.int64, count=n)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=indptr[1:])
    if indptr[-1] == 0:
        return indptr, np.zeros(0, dtype=np.int32)
    try:  # (1-D arrays / lists: one concatenate, no per-row conversion)
        flat = np.concatenate(positives).astype(np.int64, copy=False)
    except ValueError:
        flat = np.concatenate([np.asarray(p, dtype=np.int64).ravel() for p in positives])
    if flat.ndim != 1 or flat.size != indptr[-1]:
        flat = np.concatenate([np.asarray(p, dtype=np.int64).ravel() for p in positives])
    row = None
    inner = np.ones(max(flat.size - 1, 0), dtype=bool)  # adjacent pairs inside one row
    b = indptr[1:-1]
    inner[b[(b > 0) & (b < flat.size)] - 1] = False
    step = np.diff(flat)
    if (step[inner] < 0).any():
        row = np.repeat(np.arange(n, dtype=np.int64), lens)
        flat = flat[np.lexsort((flat, row))]
        step = np.diff(flat)
    if unique and (step[inner] == 0).any():
        if row is None:
            row = np.repeat(np.arange(n, dtype=np.int64), lens)
        keep = np.ones(flat.size, dtype=bool)
        keep[1:] = ~((step == 0) & inner)
        flat, row = flat[keep], row[keep]
        np.cumsum(np.bincount(row, minlength=n), out=indptr[1:])
    return indptr, flat.astype(np.int32)


def retrieve_hard_negatives(index, embeddings, positives, k_h: int, query_beam: int = 128,
                            mode: str | None = None) -> NegativeCache:
    """Per query: top (k_h + |positives|), drop the positives, keep k_h
    (anns.py:233-268), ids int32, descending score, ties to the lower id."""
    N = embeddings.shape[0]
    if k_h == 0:
        return NegativeCache(np.empty((N, 0), dtype=np.int32), index.snapshot_epoch)
    max_pos = max((len(p) for p in positives), default=0)
    if k_h + max_pos > index.size:
        raise ConfigError("k_h plus the positive count exceeds the label count")
    if index.kind != "exact":
        if _approx_impl is None:
            raise ConfigError(f"index kind {index.kind!r} is not served by the B200 refresh")
        return _approx_impl(index, embeddings, positives, k_h, query_beam)
    ops = _backend.get()
    L, d = index.vectors.shape
    mode = mode or refresh_mode_for(d, L)
    labels = _device_snapshot(index, mode)
    dev = labels["labels_f32"].device
    E = np.ascontiguousarray(embeddings, dtype=np.float32)
    out = np.empty((N, k_h), dtype=np.int32)
    for lo in range(0, N, QUERY_CHUNK):
        hi = min(N, lo + QUERY_CHUNK)
        indptr, ids = positives_csr(positives[lo:hi])
        _, top, _ = ops.refresh_topk(
            torch.from_numpy(E[lo:hi]).to(dev), torch.from_numpy(indptr).to(dev), torch.from_numpy(ids).to(dev),
            k_h, mode, **labels)
        out[lo:hi] = top.cpu().numpy()
    return NegativeCache(out, index.snapshot_epoch)


def query_topk_batch(index, queries, k: int, mode: str | None = None):
    """Exact top-k (ids int64, scores float64) of every query row against the
    index, descending, ties toward the lower id, no exclusions: the same fused
    refresh kernel with empty positive lists. fp32-exact (sequential fmaf) by
    default, so ids follow the reference's float64 ranking up to fp32 ties."""
    if index.kind != "exact":
        raise ConfigError("query_topk_batch serves exact indexes")
    if k > index.size:
        raise ConfigError(f"k={k} exceeds index size {index.size}")
    ops = _backend.get()
    L, d = index.vectors.shape
    mode = mode or os.environ.get("ASTRA_QUERY_MODE", "fp32")
    labels = _device_snapshot(index, mode)
    dev = labels["labels_f32"].device
    Q = np.ascontiguousarray(np.atleast_2d(queries), dtype=np.float32)
    N = Q.shape[0]
    ids = np.empty((N, k), dtype=np.int64)
    scores = np.empty((N, k), dtype=np.float64)
    for lo in range(0, N, QUERY_CHUNK):
        hi = min(N, lo + QUERY_CHUNK)
        indptr = torch.zeros(hi - lo + 1, dtype=torch.int64, device=dev)
        pid = torch.zeros(0, dtype=torch.int32, device=dev)
        _, top, sc = ops.refresh_topk(torch.from_numpy(Q[lo:hi]).to(dev), indptr, pid, k, mode, **labels)
        ids[lo:hi] = top.cpu().numpy()
        scores[lo:hi] = sc.cpu().numpy()
    return ids, scores


def query_topk(index, query, k: int, query_beam: int = 128):
    """Top-k ids by inner product for one query (anns.py:211-230); exact
    indexes on the GPU, graph indexes through the reference implementation."""
    if index.kind != "exact":
        if _approx_query_impl is None:
            raise ConfigError(f"index kind {index.kind!r} is not served by the B200 path")
        return _approx_query_impl(index, query, k, query_beam)
    ids, scores = query_topk_batch(index, np.asarray(query, dtype=np.float64)[None, :], k)
    return ScoredLabels(ids[0], scores[0])
