"""The importance-sampled class end to end on the GPU (PAPER.md:181-189,
SURVEY §8c "parity-unpinned extensions"): a stale refresh of top-(k_h + n_c)
-> astra_importance_split (H, candidates C, q = sigmoid(stale score)) ->
Philox draws with weight 1/(k_i q) -> the fused sampled loss. There is no
reference implementation; the contract is unbiasedness: the mean of the
sampled loss equals the full BCE loss over all labels (loss.py:67-75), the
harness of test_acceptance.py:144-187 / test_oracle_c.py applied here to the
CUDA path, and the split / draws equal the oracle restatement."""

import numpy as np
import pytest
import torch

from gpu_util import csr
from oracle import c_oracle as co
from oracle import xcmix_port as port

pytestmark = pytest.mark.gpu


def test_importance_split_matches_numpy(cuda_lib):
    from paper_2409_20156_b200 import ops

    rng = np.random.default_rng(1)
    nq, k_h, n_c = 300, 7, 13
    ids = rng.integers(0, 10_000, size=(nq, k_h + n_c)).astype(np.int32)
    ids[5, -3:] = -1  # fewer labels than asked
    scores = (rng.standard_normal((nq, k_h + n_c)) * 4).astype(np.float32)
    hard, cand, q = ops.importance_split(torch.from_numpy(ids).cuda(), torch.from_numpy(scores).cuda(), k_h)
    np.testing.assert_array_equal(hard.cpu().numpy(), ids[:, :k_h])
    np.testing.assert_array_equal(cand.cpu().numpy(), ids[:, k_h:])
    ref = (1.0 / (1.0 + np.exp(-scores[:, k_h:].astype(np.float64)))).astype(np.float32)
    ref[ids[:, k_h:] < 0] = 0.0
    np.testing.assert_allclose(q.cpu().numpy(), ref, rtol=2e-7, atol=0)


def test_engine_importance_mixture_unbiased(cuda_lib):
    """E[sampled loss] == full BCE (Monte Carlo over Philox draws), through
    ClassifierEngine: refresh_cache -> sample(k_i > 0) -> step (lr = 0)."""
    from paper_2409_20156_b200.engine import ClassifierEngine

    rng = np.random.default_rng(5)
    L, d, k_p, k_h, n_c, k_i, k_r = 3000, 64, 2, 8, 40, 16, 64
    W = rng.uniform(-0.3, 0.3, size=(L, d)).astype(np.float32)
    eng = ClassifierEngine(L, d, k_p=k_p, k_h=k_h, k_r=k_r, k_i=k_i, n_c=n_c, weights=W, refresh_mode="fp32", seed=3)
    eng.snapshot(0)
    q = rng.standard_normal(d).astype(np.float32)
    pos = np.array([17, 2500], np.int32)  # |P| <= k_p: every positive is in every slate
    ip, pid = csr([pos])
    hard, cand, cand_q = eng.refresh_cache(torch.from_numpy(q[None]).cuda(), torch.from_numpy(ip).cuda(),
                                           torch.from_numpy(pid).cuda())
    # the cache equals the fp32 oracle's top-(k_h + n_c) split
    _, oids, oscores = co.refresh_fp32(q[None], W, ip, pid, k_h + n_c)
    np.testing.assert_array_equal(hard.cpu().numpy(), oids[:, :k_h])
    np.testing.assert_array_equal(cand.cpu().numpy(), oids[:, k_h:])
    s_all = (W.astype(np.float64) @ q.astype(np.float64))
    full = float(port.softplus64(-s_all[pos]).sum() + port.softplus64(np.delete(s_all, pos)).sum())
    B, n_batches = 2048, 40
    emb = torch.from_numpy(np.tile(q, (B, 1))).cuda()
    ipB, pidB = csr([pos] * B)
    ipB, pidB = torch.from_numpy(ipB).cuda(), torch.from_numpy(pidB).cuda()
    H, C, Q = hard.expand(B, -1).contiguous(), cand.expand(B, -1).contiguous(), cand_q.expand(B, -1).contiguous()
    means = []
    for t in range(n_batches):
        rows = torch.arange(t * B, (t + 1) * B, dtype=torch.int64, device="cuda")
        slates = eng.sample(rows, ipB, pidB, H, epoch=1, step=t, cand=C, cand_q=Q)
        if t == 0:  # draws equal the oracle sampler's, draw for draw
            ref = co.sample_slates(eng.seed, 1, 0, rows.cpu().numpy(), ipB.cpu().numpy(), pidB.cpu().numpy(),
                                   H.cpu().numpy(), k_h, L, k_p, k_r, cand=C.cpu().numpy(), cand_q=Q.cpu().numpy(),
                                   k_i=k_i)
            for g_, r_ in zip(slates, ref):
                np.testing.assert_array_equal(g_.cpu().numpy(), r_)
        loss, _, status = eng.step(emb, slates, 0.0, 0.0)
        assert not status.cpu().numpy().any()
        means.append(float(loss.item()) / B)
    np.testing.assert_array_equal(eng.W.cpu().numpy(), W)  # lr = 0: W untouched
    est = float(np.mean(means))
    se = float(np.std(means) / np.sqrt(len(means)))
    print(f"importance mixture: estimate {est:.4f} +- {se:.4f}, full loss {full:.4f}")
    assert abs(est - full) < 4 * se + 1e-6 * abs(full)
