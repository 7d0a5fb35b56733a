"""Helpers shared by the -m gpu tests (host<->device conversions)."""

import numpy as np
import torch


def dev(a, dtype=None):
    t = torch.as_tensor(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def csr(positives):
    indptr = np.zeros(len(positives) + 1, np.int64)
    indptr[1:] = np.cumsum([len(p) for p in positives])
    ids = np.concatenate([np.asarray(p, np.int32) for p in positives]) if len(positives) else np.zeros(0, np.int32)
    return indptr, ids.astype(np.int32)


def random_positives(rng, n, L, lo=0, hi=5):
    return [np.sort(rng.choice(L, size=int(rng.integers(lo, hi + 1)), replace=False)).astype(np.int32) for _ in range(n)]


def u64(t):
    return t.cpu().numpy().view(np.uint64)
