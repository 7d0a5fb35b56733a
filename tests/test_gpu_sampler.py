"""GPU Philox sampler == C oracle sampler draw-for-draw (integer work: bit-exact).

The oracle's distributional contract is pinned in tests/test_oracle_c.py
(restating the reference's sampler tests), so bit-equality transfers it."""

import numpy as np
import pytest
import torch

from gpu_util import csr, dev
from oracle import c_oracle as co

pytestmark = pytest.mark.gpu


def _case(seed, B, L, k_p, k_h, k_r, k_i=0, n_c=0, pos_hi=8):
    rng = np.random.default_rng(seed)
    positives = [np.sort(rng.choice(L, size=int(rng.integers(0, pos_hi + 1)), replace=False)).astype(np.int32) for _ in range(B)]
    hard = cand = q = None
    if k_h or n_c:
        hard_all = np.stack([rng.choice(np.setdiff1d(np.arange(L), positives[b]), size=k_h + n_c, replace=False)
                             for b in range(B)]).astype(np.int32)
        hard = np.ascontiguousarray(hard_all[:, :k_h]) if k_h else None
        if n_c:
            cand = np.ascontiguousarray(hard_all[:, k_h:])
            q = rng.uniform(0.05, 1.0, size=cand.shape).astype(np.float32)
    rows = rng.integers(0, 1 << 31, size=B).astype(np.int64)
    return positives, hard, cand, q, rows


@pytest.mark.parametrize("B,L,k_p,k_h,k_r,k_i,n_c", [
    (64, 1000, 3, 16, 16, 0, 0),        # C1-like
    (37, 700, 4, 0, 16, 0, 0),          # warm phase: no hard slots
    (16, 131073, 8, 64, 512, 0, 0),     # C2 slate
    (20, 5000, 2, 10, 30, 12, 40),      # importance extension
    (8, 60, 5, 20, 7, 0, 0),            # heavy padding, small L
])
def test_sampler_matches_oracle(cuda_lib, B, L, k_p, k_h, k_r, k_i, n_c):
    from paper_2409_20156_b200 import ops

    positives, hard, cand, q, rows = _case(B + L, B, L, k_p, k_h, k_r, k_i, n_c)
    ip, pid = csr(positives)
    ref = co.sample_slates(1234, 5, 77, rows, ip, pid, hard, k_h, L, k_p, k_r, cand=cand, cand_q=q, k_i=k_i)
    got = ops.sample_slates(1234, 5, 77, dev(rows), dev(ip), dev(pid), None if hard is None else dev(hard), k_h, L,
                            k_p, k_r, cand=None if cand is None else dev(cand), cand_q=None if q is None else dev(q),
                            k_i=k_i)
    torch.cuda.synchronize()
    for r, g in zip(ref, got):
        np.testing.assert_array_equal(g.cpu().numpy(), r)


def test_sampler_infeasible(cuda_lib):
    from paper_2409_20156_b200 import ops
    from paper_2409_20156_b200.errors import ConfigError

    rows = dev(np.arange(2, dtype=np.int64))
    ip = dev(np.zeros(3, np.int64))
    pid = dev(np.zeros(0, np.int32))
    hard = dev(np.array([[0, 1, 2], [0, 1, 2]], np.int32))
    with pytest.raises(ConfigError):
        ops.sample_slates(0, 0, 0, rows, ip, pid, hard, 3, 3, 1, 1)  # sampler.py:120-121
