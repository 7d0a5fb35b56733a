"""astra_gemm_f32 (3xTF32 on the tf32 tensor cores), the all-negatives arm's
GEMMs (trainer.py:593-606: E W^T, G W, G^T E). fp32 accuracy: every entry
within 1e-5 of the float64 product relative to sum_k |a_ik b_jk| (the
conditioning-aware form of the north star's 1e-5 fp32 tolerance; an fp32
sgemm's own rounding is ~K * 2^-24 of the same quantity)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _check(D, A, B):
    A64, B64 = A.astype(np.float64), B.astype(np.float64)
    ref = A64 @ B64.T
    scale = np.abs(A64) @ np.abs(B64).T
    err = np.abs(D.astype(np.float64) - ref)
    worst = float((err / np.maximum(scale, 1e-30)).max())
    assert worst <= 1e-5, worst
    return worst


@pytest.mark.parametrize("M,N,K,a_t,b_t", [
    (1024, 50_000, 768, False, False),   # scores = E W^T (the arm's first GEMM)
    (1024, 768, 50_000, False, True),    # grad_emb = G W (split-K)
    (50_000, 768, 1024, True, True),     # grad_W = G^T E
    (100, 37, 5, False, False),          # ragged tiles, K < 32
    (300, 513, 1000, True, False),
    (7, 1, 64, False, True),
])
def test_gemm_f32_matches_float64(cuda_lib, M, N, K, a_t, b_t):
    from paper_2409_20156_b200 import ops

    rng = np.random.default_rng(M + N + K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = (rng.standard_normal((N, K)) * rng.uniform(0.01, 10, size=(N, 1))).astype(np.float32)
    a_in = np.ascontiguousarray(A.T) if a_t else A
    b_in = np.ascontiguousarray(B.T) if b_t else B
    D = ops.gemm_f32(torch.from_numpy(a_in).cuda(), torch.from_numpy(b_in).cuda(), a_t=a_t, b_t=b_t)
    torch.cuda.synchronize()
    if M * N > 4_000_000:  # the float64 reference on a row sample
        rows = np.sort(rng.choice(M, size=64, replace=False))
        worst = _check(D[torch.from_numpy(rows).cuda()].cpu().numpy(), A[rows], B)
    else:
        worst = _check(D.cpu().numpy(), A, B)
    print(f"[gemm_f32 {M}x{N}x{K}] worst error / sum|a||b| = {worst:.2e}")


def test_gemm_f32_beats_plain_tf32(cuda_lib):
    """The split matters: a single tf32 product would miss the bar by ~100x."""
    from paper_2409_20156_b200 import ops

    rng = np.random.default_rng(1)
    A = rng.standard_normal((256, 512)).astype(np.float32)
    B = rng.standard_normal((256, 512)).astype(np.float32)
    D = ops.gemm_f32(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()).cpu().numpy()
    tf = lambda x: (x.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32).astype(np.float64)  # noqa: E731
    plain = tf(A) @ tf(B).T
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    scale = np.abs(A.astype(np.float64)) @ np.abs(B.astype(np.float64)).T
    assert (np.abs(plain - ref) / scale).max() > 1e-4
    assert (np.abs(D - ref) / scale).max() < 1e-5
