"""ctypes binding of oracle/_build/libastra_oracle.so — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may use
this module. See oracle/astra_oracle.c for what the restatement covers.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libastra_oracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = ctypes.CDLL(LIB_PATH)
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def refresh_fp32(Q, W, pos_indptr, pos_ids, k, label_offset=0):
    """Exact fixed-order fp32 refresh: (keys, ids, scores), each nq x k."""
    lib = load()
    Q = np.ascontiguousarray(Q, np.float32)
    W = np.ascontiguousarray(W, np.float32)
    pos_indptr = np.ascontiguousarray(pos_indptr, np.int64)
    pos_ids = np.ascontiguousarray(pos_ids, np.int32)
    nq, d = Q.shape
    keys = np.zeros((nq, k), np.uint64)
    ids = np.zeros((nq, k), np.int32)
    scores = np.zeros((nq, k), np.float32)
    lib.oracle_refresh_fp32(
        _p(Q), ctypes.c_int64(nq), ctypes.c_int(d), _p(W), ctypes.c_int64(W.shape[0]), ctypes.c_int64(label_offset),
        _p(pos_indptr), _p(pos_ids), ctypes.c_int(k), _p(keys), _p(ids), _p(scores),
    )
    return keys, ids, scores


def refresh_fp32_blocked(Q, W, pos_indptr, pos_ids, k, label_offset=0, nthreads=0):
    """The same keys as refresh_fp32 (identical fmaf chains), blocked and
    threaded for production-size checks. W: fp32, or bf16 given as a uint16 /
    int16 array of bit patterns (widened exactly, as the re-rank does)."""
    lib = load()
    Q = np.ascontiguousarray(Q, np.float32)
    W = np.ascontiguousarray(W)
    if W.dtype in (np.uint16, np.int16):
        w_bf16 = 1
    else:
        W = np.ascontiguousarray(W, np.float32)
        w_bf16 = 0
    pos_indptr = np.ascontiguousarray(pos_indptr, np.int64)
    pos_ids = np.ascontiguousarray(pos_ids, np.int32)
    nq, d = Q.shape
    keys = np.zeros((nq, k), np.uint64)
    ids = np.zeros((nq, k), np.int32)
    scores = np.zeros((nq, k), np.float32)
    lib.oracle_refresh_fp32_blocked(
        _p(Q), ctypes.c_int64(nq), ctypes.c_int(d), _p(W), ctypes.c_int(w_bf16), ctypes.c_int64(W.shape[0]),
        ctypes.c_int64(label_offset), _p(pos_indptr), _p(pos_ids), ctypes.c_int(k), ctypes.c_int(nthreads),
        _p(keys), _p(ids), _p(scores),
    )
    return keys, ids, scores


def scores_fp32(Q, W):
    lib = load()
    Q = np.ascontiguousarray(Q, np.float32)
    W = np.ascontiguousarray(W, np.float32)
    out = np.empty((Q.shape[0], W.shape[0]), np.float32)
    lib.oracle_scores_fp32(_p(Q), ctypes.c_int64(Q.shape[0]), ctypes.c_int(Q.shape[1]), _p(W), ctypes.c_int64(W.shape[0]), _p(out))
    return out


def philox4x32_10(ctr, key):
    lib = load()
    c = np.ascontiguousarray(ctr, np.uint32)
    k = np.ascontiguousarray(key, np.uint32)
    out = np.zeros(4, np.uint32)
    lib.oracle_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def sample_slates(seed, epoch, step, rows, pos_indptr, pos_ids, hard, k_h, n_labels, k_p, k_r,
                  cand=None, cand_q=None, k_i=0):
    """Philox slates (ids, y, origin, weights), each B x S — the spec the GPU
    sampler must match draw-for-draw."""
    lib = load()
    rows = np.ascontiguousarray(rows, np.int64)
    B = len(rows)
    pos_indptr = np.ascontiguousarray(pos_indptr, np.int64)
    pos_ids = np.ascontiguousarray(pos_ids, np.int32)
    if hard is None or k_h == 0:
        hard = np.zeros((B, 1), np.int32)
        k_h = 0
    hard = np.ascontiguousarray(hard, np.int32)
    n_c = 0
    cand_stride = 1
    if cand is not None and k_i > 0:
        cand = np.ascontiguousarray(cand, np.int32)
        cand_q = np.ascontiguousarray(cand_q, np.float32)
        n_c = cand.shape[1]
        cand_stride = n_c
    else:
        k_i = 0
    S = k_p + k_h + k_i + k_r
    ids = np.zeros((B, S), np.int32)
    y = np.zeros((B, S), np.int8)
    origin = np.zeros((B, S), np.int8)
    weights = np.zeros((B, S), np.float32)
    rc = lib.oracle_sample_slates(
        ctypes.c_uint64(seed), ctypes.c_uint32(epoch), ctypes.c_uint32(step), _p(rows), ctypes.c_int(B),
        _p(pos_indptr), _p(pos_ids), _p(hard), ctypes.c_int(hard.shape[1]), ctypes.c_int(k_h),
        _p(cand), _p(cand_q), ctypes.c_int(cand_stride), ctypes.c_int(n_c), ctypes.c_int(k_i),
        ctypes.c_int64(n_labels), ctypes.c_int(k_p), ctypes.c_int(k_r), _p(ids), _p(y), _p(origin), _p(weights),
    )
    if rc != 0:
        raise ValueError("infeasible sampler configuration")
    return ids, y, origin, weights


def key_to_score(keys):
    o = (np.asarray(keys, np.uint64) >> np.uint64(32)).astype(np.uint32)
    b = np.where(o & np.uint32(0x80000000), o & np.uint32(0x7FFFFFFF), ~o).astype(np.uint32)
    return b.view(np.float32)


def key_to_id(keys):
    return (np.uint32(0xFFFFFFFF) - (np.asarray(keys, np.uint64) & np.uint64(0xFFFFFFFF)).astype(np.uint32)).astype(np.int32)
