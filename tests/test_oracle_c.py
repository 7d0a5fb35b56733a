"""Pin the C oracle (oracle/astra_oracle.c): Philox known answers, the fixed-
order fp32 refresh against the reference's golden ids, and the sampler's
distributional contract restated from the reference's sampler tests."""

import numpy as np
import pytest

from conftest import golden
from oracle import c_oracle as co
from oracle import xcmix_port as port


def _csr(positives):
    indptr = np.zeros(len(positives) + 1, np.int64)
    indptr[1:] = np.cumsum([len(p) for p in positives])
    ids = np.concatenate([np.asarray(p, np.int32) for p in positives]) if positives else np.zeros(0, np.int32)
    return indptr, ids.astype(np.int32)


def test_philox_known_answers():
    # Random123 philox4x32-10 known-answer vectors (kat_vectors).
    assert co.philox4x32_10([0, 0, 0, 0], [0, 0]).tolist() == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert co.philox4x32_10([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2).tolist() == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert co.philox4x32_10([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0]).tolist() == [
        0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


def test_refresh_ties_fixture_exact():
    # grid-valued inputs: every summation order gives the same fp32 scores, so
    # the fixed-order restatement must equal the reference bit-for-bit
    g = golden("refresh_ties.npz")
    _, ids, _ = co.refresh_fp32(g["E"], g["W"], g["pos_indptr"], g["pos_ids"], int(g["k_h"]))
    np.testing.assert_array_equal(ids, g["ids"])


def test_refresh_random_fixture_up_to_ties():
    g = golden("refresh_random.npz")
    k = int(g["k_h"])
    _, ids, scores = co.refresh_fp32(g["E"], g["W"], g["pos_indptr"], g["pos_ids"], k)
    ref = g["ids"]
    full = co.scores_fp32(g["E"], g["W"])
    diff = ids != ref
    # ids only differ where sgemm vs fixed-order rounding swaps near-equal scores
    for i, j in zip(*np.nonzero(diff)):
        assert abs(full[i, ids[i, j]] - full[i, ref[i, j]]) < 1e-5
    assert diff.mean() < 0.01


@pytest.mark.parametrize("nq,L,d,k,offset", [(37, 5003, 64, 20, 0), (16, 2048, 768, 64, 1000), (5, 3, 8, 6, 0),
                                             (50, 20000, 24, 200, 7)])
def test_refresh_blocked_equals_scalar(nq, L, d, k, offset):
    # the blocked/threaded/vectorised oracle used by the production-size GPU
    # parity tests computes the same fmaf chains: keys bit-identical
    rng = np.random.default_rng(nq * 7 + L)
    W = rng.standard_normal((L, d)).astype(np.float32)
    Q = rng.standard_normal((nq, d)).astype(np.float32)
    Q[1 % nq] = 0.0  # an all-tie query
    positives = [np.sort(rng.choice(L, size=int(rng.integers(0, min(L, 6))), replace=False)) + offset for _ in range(nq)]
    ip, pid = _csr(positives)
    ref = co.refresh_fp32(Q, W, ip, pid, k, label_offset=offset)
    for nth in (1, 3):
        got = co.refresh_fp32_blocked(Q, W, ip, pid, k, label_offset=offset, nthreads=nth)
        for a, b in zip(got, ref):
            np.testing.assert_array_equal(a, b)


def test_refresh_blocked_bf16_rows():
    # bf16 W as bit patterns = the fp32 oracle on the widened values
    rng = np.random.default_rng(5)
    W = rng.standard_normal((3000, 128)).astype(np.float32)
    bits = (W.view(np.uint32) >> 16).astype(np.uint16)
    Wb = (bits.astype(np.uint32) << 16).view(np.float32)
    Q = rng.standard_normal((20, 128)).astype(np.float32)
    ip, pid = _csr([np.zeros(0, np.int32)] * 20)
    a = co.refresh_fp32_blocked(Q, bits, ip, pid, 50)
    b = co.refresh_fp32(Q, Wb, ip, pid, 50)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


def test_refresh_reference_known_answers():
    W = np.array([[0.0, 1.0], [1.0, 0.0], [1.0, 0.0], [0.5, 0.0]], np.float32)
    _, ids, _ = co.refresh_fp32(np.array([[1.0, 0.0]], np.float32), W, [0, 0], [], 3)
    assert ids[0].tolist() == [1, 2, 3]  # test_anns.py:30-33
    W = np.random.default_rng(1).standard_normal((20, 4)).astype(np.float32)
    _, ids, _ = co.refresh_fp32(np.zeros((1, 4), np.float32), W, [0, 0], [], 5)
    assert ids[0].tolist() == [0, 1, 2, 3, 4]  # test_anns.py:46-50
    # positives excluded, label offset applied (shard view)
    _, ids, _ = co.refresh_fp32(np.zeros((1, 4), np.float32), W, [0, 2], [101, 103], 3, label_offset=100)
    assert ids[0].tolist() == [100, 102, 104]


def test_refresh_matches_port_on_random():
    rng = np.random.default_rng(5)
    W = rng.standard_normal((400, 24)).astype(np.float32)
    E = rng.standard_normal((40, 24)).astype(np.float32)
    positives = [np.sort(rng.choice(400, size=3, replace=False)).astype(np.int32) for _ in range(40)]
    ip, pid = _csr(positives)
    _, ids, _ = co.refresh_fp32(E, W, ip, pid, 12)
    ref = port.retrieve_hard_negatives(W, E, positives, 12)
    full = co.scores_fp32(E, W)
    for i, j in zip(*np.nonzero(ids != ref)):
        assert abs(full[i, ids[i, j]] - full[i, ref[i, j]]) < 1e-5


# ---------------------------------------------------------------- sampler


def _sample(B=64, L=100, k_p=3, k_h=5, k_r=40, seed=0, npos=None, hard=None, **kw):
    rng = np.random.default_rng(seed)
    positives = []
    for b in range(B):
        n = int(rng.integers(0, 6)) if npos is None else npos
        positives.append(np.sort(rng.choice(L, size=n, replace=False)).astype(np.int32))
    if hard is None and k_h:
        hard = np.stack([rng.choice(np.setdiff1d(np.arange(L), positives[b]), size=k_h, replace=False) for b in range(B)]).astype(np.int32)
    ip, pid = _csr(positives)
    out = co.sample_slates(seed, 3, 7, np.arange(B) + 1000, ip, pid, hard, k_h, L, k_p, k_r, **kw)
    return positives, hard, out


def test_sampler_structure():
    positives, hard, (ids, y, origin, w) = _sample()
    k_p, k_h, L = 3, 5, 100
    for b in range(len(positives)):
        P = set(positives[b].tolist())
        np_ = min(len(P), k_p)
        assert set(ids[b, :np_].tolist()) <= P and (y[b, :np_] == 1).all() and (origin[b, :np_] == 0).all()
        assert (origin[b, np_:k_p] == 3).all() and (y[b, np_:k_p] == 0).all()
        assert not set(ids[b, np_:k_p].tolist()) & P  # pads avoid positives
        assert ids[b, k_p : k_p + k_h].tolist() == hard[b].tolist()
        rand = ids[b, k_p + k_h :]
        assert not set(rand.tolist()) & set(hard[b].tolist())  # complement of H
        assert ((rand >= 0) & (rand < L)).all()
        assert y[b, k_p + k_h :].tolist() == [int(r in P) for r in rand]
        np.testing.assert_array_equal(w[b, k_p + k_h :], np.float32((L - k_h) / 40))
        assert (w[b, : k_p + k_h] == 1.0).all()


def test_sampler_deterministic_and_keyed():
    a = _sample(seed=1)[2]
    b = _sample(seed=1)[2]
    for x, z in zip(a, b):
        np.testing.assert_array_equal(x, z)
    positives, hard, _ = _sample(seed=1)
    ip, pid = _csr(positives)
    c = co.sample_slates(1, 3, 8, np.arange(64) + 1000, ip, pid, hard, 5, 100, 3, 40)
    assert not np.array_equal(a[0], c[0])  # a different step draws differently


def test_sampler_marginal_frequency():
    # restates test_sampler.py:122-132: uniform over [L] \ H within 5 sigma
    L, B, k_r = 100, 400, 250
    hard = np.tile(np.arange(10, dtype=np.int32), (B, 1))
    _, _, (ids, _, _, _) = _sample(B=B, L=L, k_p=1, k_h=10, k_r=k_r, npos=0, hard=hard, seed=2)
    draws = ids[:, 11:].ravel()
    p = 1.0 / 90.0
    tol = 5 * np.sqrt(p * (1 - p) / draws.size)
    assert draws.min() >= 10
    for lab in (10, 47, 99):
        assert abs((draws == lab).mean() - p) < tol
    counts = np.bincount(draws, minlength=L)[10:]
    chi2 = ((counts - draws.size * p) ** 2 / (draws.size * p)).sum()
    assert chi2 < 89 + 6 * np.sqrt(2 * 89)  # chi-square over all 90 labels


def test_sampler_forced_complement_and_replacement():
    # test_sampler.py:105-120
    hard = np.tile(np.arange(10, dtype=np.int32), (4, 1))
    _, _, (ids, _, _, _) = _sample(B=4, L=12, k_p=1, k_h=10, k_r=10, npos=0, hard=hard)
    rand = ids[:, 11:]
    assert set(rand.ravel().tolist()) <= {10, 11}
    assert len(set(rand[0].tolist())) < 10


def test_sampler_positive_subset_uniform():
    # test_sampler.py:92-101: k_p-subsets of 10 positives are uniform
    B, L = 6000, 50
    pos = [np.arange(10, dtype=np.int32)] * B
    ip, pid = _csr(pos)
    ids, y, _, _ = co.sample_slates(4, 0, 0, np.arange(B), ip, pid, None, 0, L, 3, 1)
    sub = ids[:, :3]
    assert all(len(set(r)) == 3 for r in sub.tolist())
    freq = np.bincount(sub.ravel(), minlength=10)[:10] / sub.size
    assert np.abs(freq - 0.1).max() < 0.01


def test_sampler_importance_weights_unbiased():
    """Importance extension: E[estimator] == full BCE loss (Monte Carlo),
    the harness of test_acceptance.py:144-187 applied to the H + I + R mixture."""
    rng = np.random.default_rng(9)
    L, d, k_h, n_c, k_i, k_r = 120, 8, 4, 12, 6, 10
    Wm = rng.standard_normal((L, d))
    emb = rng.standard_normal(d)
    s_all = Wm @ emb
    pos = np.array([3, 77], np.int32)
    full = float(port.softplus64(-s_all[pos]).sum() + port.softplus64(np.delete(s_all, pos)).sum())
    order = [l for l in np.lexsort((np.arange(L), -s_all)) if l not in pos]
    hard = np.array(order[:k_h], np.int32)
    cand = np.array(order[k_h : k_h + n_c], np.int32)
    q = (1.0 / (1.0 + np.exp(-s_all[cand]))).astype(np.float32)
    T = 4000
    ip, pid = _csr([pos] * T)
    ids, y, origin, w = co.sample_slates(11, 0, 0, np.arange(T), ip, pid, np.tile(hard, (T, 1)), k_h, L, 2, k_r,
                                         cand=np.tile(cand, (T, 1)), cand_q=np.tile(q, (T, 1)), k_i=k_i)
    s = s_all[ids]
    loss, _ = port.slate_factors(s.astype(np.float64), y, origin, w)
    per = np.array([port.slate_factors(s[t : t + 1].astype(np.float64), y[t : t + 1], origin[t], w[t])[0] for t in range(0, T, 40)])
    est = loss / T
    se = per.std() / np.sqrt(len(per)) * np.sqrt(len(per) / T)
    assert abs(est - full) < 4 * se + 1e-9
