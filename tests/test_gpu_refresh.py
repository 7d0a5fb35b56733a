"""GPU parity of the shortlist refresh (anns.py:233-256) through the C-ABI.

FP32_EXACT ids/keys must equal the C oracle bit-for-bit; BF16_RERANK must
equal FP32_EXACT; plain BF16 must reach the recall bar against fp32.
"""

import os
import numpy as np
import pytest
import torch

from conftest import golden
from gpu_util import csr, dev, random_positives, u64
from oracle import c_oracle as co

pytestmark = pytest.mark.gpu


def _run(E, W, positives, k, mode, offset=0):
    from paper_2409_20156_b200 import ops

    ip, pid = csr(positives)
    Wd = dev(W)
    extra = {"labels_e4m3": ops.quantize_e4m3(Wd)} if mode == "fp8_rerank" else {}
    keys, ids, scores = ops.refresh_topk(
        dev(E), dev(ip), dev(pid), k, mode, labels_f32=Wd,
        labels_bf16=ops.f32_to_bf16(Wd) if mode in ("bf16", "bf16_rerank") else None, label_offset=offset, **extra)
    torch.cuda.synchronize()
    return u64(keys), ids.cpu().numpy(), scores.cpu().numpy()


@pytest.mark.parametrize("name", ["refresh_random.npz", "refresh_ties.npz"])
def test_fp32_exact_matches_oracle_on_golden(cuda_lib, name):
    g = golden(name)
    ip, pid = g["pos_indptr"], g["pos_ids"]
    positives = [pid[ip[i] : ip[i + 1]] for i in range(len(ip) - 1)]
    k = int(g["k_h"])
    keys, ids, _ = _run(g["E"], g["W"], positives, k, "fp32")
    okeys, oids, _ = co.refresh_fp32(g["E"], g["W"], ip, pid, k)
    np.testing.assert_array_equal(keys, okeys)
    np.testing.assert_array_equal(ids, oids)
    if name == "refresh_ties.npz":  # order-independent scores: equals the reference itself
        np.testing.assert_array_equal(ids, g["ids"])


@pytest.mark.parametrize("nq,L,d,k", [(130, 1000, 24, 5), (257, 5000, 64, 64), (64, 3000, 96, 300), (33, 700, 128, 600)])
def test_fp32_exact_shapes(cuda_lib, nq, L, d, k):
    rng = np.random.default_rng(nq + L)
    W = rng.standard_normal((L, d)).astype(np.float32)
    E = rng.standard_normal((nq, d)).astype(np.float32)
    positives = random_positives(rng, nq, L, 0, 6)
    keys, ids, scores = _run(E, W, positives, k, "fp32")
    okeys, oids, oscores = co.refresh_fp32(E, W, *csr(positives), k)
    np.testing.assert_array_equal(keys, okeys)
    np.testing.assert_array_equal(ids, oids)
    np.testing.assert_array_equal(scores, oscores)


def test_known_answers(cuda_lib):
    W = np.array([[0.0, 1.0], [1.0, 0.0], [1.0, 0.0], [0.5, 0.0]], np.float32)
    _, ids, _ = _run(np.array([[1.0, 0.0]], np.float32), W, [np.zeros(0, np.int32)], 3, "fp32")
    assert ids[0].tolist() == [1, 2, 3]  # test_anns.py:30-33
    W = np.random.default_rng(1).standard_normal((20, 4)).astype(np.float32)
    _, ids, _ = _run(np.zeros((1, 4), np.float32), W, [np.zeros(0, np.int32)], 5, "fp32")
    assert ids[0].tolist() == [0, 1, 2, 3, 4]  # test_anns.py:46-50


def test_shard_merge_equals_single_shard(cuda_lib):
    from paper_2409_20156_b200 import ops

    rng = np.random.default_rng(3)
    L, d, nq, k = 6000, 64, 200, 40
    W = rng.standard_normal((L, d)).astype(np.float32)
    E = rng.standard_normal((nq, d)).astype(np.float32)
    positives = random_positives(rng, nq, L, 0, 8)
    full_keys, full_ids, _ = _run(E, W, positives, k, "fp32")
    bounds = [0, 1700, 4100, L]
    parts = []
    for lo, hi in zip(bounds[:-1], bounds[1:]):
        keys, _, _ = _run(E, W[lo:hi], positives, k, "fp32", offset=lo)
        parts.append(keys)
    part_keys = dev(np.stack(parts).view(np.int64))
    mk, mids, _ = ops.topk_merge(part_keys, k)
    np.testing.assert_array_equal(u64(mk), full_keys)
    np.testing.assert_array_equal(mids.cpu().numpy(), full_ids)


@pytest.mark.parametrize("nq,L,d,k", [(256, 20000, 128, 32), (300, 9000, 768, 64), (1, 5000, 64, 8)])
def test_bf16_recall_and_rerank(cuda_lib, nq, L, d, k):
    rng = np.random.default_rng(7)
    W = rng.uniform(-1 / np.sqrt(d), 1 / np.sqrt(d), size=(L, d)).astype(np.float32)
    E = rng.standard_normal((nq, d)).astype(np.float32)
    positives = random_positives(rng, nq, L, 0, 5)
    _, exact_ids, _ = _run(E, W, positives, k, "fp32")
    _, bf_ids, bf_scores = _run(E, W, positives, k, "bf16")
    recall = np.mean([len(set(a) & set(b)) / k for a, b in zip(bf_ids.tolist(), exact_ids.tolist())])
    assert recall >= 0.98, recall
    # bf16 scores are close to the fp32 scores of the same labels
    full = co.scores_fp32(E, W)
    ref = np.take_along_axis(full, bf_ids.astype(np.int64), axis=1)
    assert np.abs(bf_scores - ref).max() < 0.05 * np.abs(full).max()
    for i, p in enumerate(positives):
        assert not set(bf_ids[i].tolist()) & set(p.tolist())
        assert len(set(bf_ids[i].tolist())) == k
    _, rr_ids, rr_scores = _run(E, W, positives, k, "bf16_rerank")
    np.testing.assert_array_equal(rr_ids, exact_ids)  # north star: recall@k >= 0.999 in bf16 mode


def test_bf16_rerank_label_offset_and_tail(cuda_lib):
    rng = np.random.default_rng(9)
    L, d, nq, k = 1000 + 37, 64, 130, 16  # label tail inside a 256-wide tile, query tail
    W = rng.standard_normal((L, d)).astype(np.float32)
    E = rng.standard_normal((nq, d)).astype(np.float32)
    positives = [p + 5000 for p in random_positives(rng, nq, L, 0, 4)]
    _, exact_ids, _ = _run(E, W, positives, k, "fp32", offset=5000)
    _, rr_ids, _ = _run(E, W, positives, k, "bf16_rerank", offset=5000)
    np.testing.assert_array_equal(rr_ids, exact_ids)
    assert rr_ids.min() >= 5000 and rr_ids.max() < 5000 + L


def test_config_errors(cuda_lib):
    from paper_2409_20156_b200 import ops
    from paper_2409_20156_b200.errors import ConfigError

    E = torch.zeros((4, 48), device="cuda")
    W = torch.zeros((10, 48), device="cuda")
    ip = torch.zeros(5, dtype=torch.int64, device="cuda")
    pid = torch.zeros(0, dtype=torch.int32, device="cuda")
    with pytest.raises(ConfigError):
        ops.refresh_topk(E, ip, pid, 3, "bf16", labels_bf16=W.to(torch.bfloat16))  # d % 64
    with pytest.raises(ConfigError):
        ops.refresh_topk(E, ip, pid, 0, "fp32", labels_f32=W)


def _with_two_pass(flag, fn):
    import os

    old = os.environ.get("ASTRA_REFRESH_TWO_PASS")
    os.environ["ASTRA_REFRESH_TWO_PASS"] = flag
    try:
        return fn()
    finally:
        if old is None:
            del os.environ["ASTRA_REFRESH_TWO_PASS"]
        else:
            os.environ["ASTRA_REFRESH_TWO_PASS"] = old


@pytest.mark.parametrize("mode,k", [("bf16", 32), ("bf16", 96), ("bf16_rerank", 64)])
@pytest.mark.parametrize("nq", [700, 2100])
def test_two_pass_equals_running_topk(cuda_lib, mode, k, nq):
    """sample -> threshold -> select -> verify must return exactly the keys of
    the single-pass running top-k (same bf16 scores), positives excluded."""
    rng = np.random.default_rng(k + nq)
    L, d = 70_000 + 129, 128  # 274 label tiles (tail inside a tile), 18 sample tiles
    W = rng.uniform(-1 / np.sqrt(d), 1 / np.sqrt(d), size=(L, d)).astype(np.float32)
    E = rng.standard_normal((nq, d)).astype(np.float32)
    positives = [p + 11 for p in random_positives(rng, nq, L, 0, 12)]  # global ids (label_offset 11)
    run_keys, run_ids, _ = _with_two_pass("0", lambda: _run(E, W, positives, k, mode, offset=11))
    tp_keys, tp_ids, _ = _with_two_pass("1", lambda: _run(E, W, positives, k, mode, offset=11))
    np.testing.assert_array_equal(tp_keys, run_keys)
    np.testing.assert_array_equal(tp_ids, run_ids)
    for i, p in enumerate(positives):
        assert not set(tp_ids[i].tolist()) & set(p.tolist())


def test_two_pass_fallback_on_adversarial_sample(cuda_lib):
    """Labels of the sampled tiles score far higher than the rest, so the
    sample threshold admits fewer than k candidates for most queries: the
    verification fallback must still give the exact result."""
    rng = np.random.default_rng(5)
    L, d, nq, k = 256 * 40, 64, 300, 48
    W = rng.uniform(-0.1, 0.1, size=(L, d)).astype(np.float32)
    E = np.abs(rng.standard_normal((nq, d))).astype(np.float32)
    for t in range(0, L // 256, 16):  # the sampled tiles (stride 16)
        W[t * 256 : (t + 1) * 256] = np.abs(W[t * 256 : (t + 1) * 256]) + 0.5
    positives = random_positives(rng, nq, L, 0, 3)
    run_keys, _, _ = _with_two_pass("0", lambda: _run(E, W, positives, k, "bf16"))
    tp_keys, _, _ = _with_two_pass("1", lambda: _run(E, W, positives, k, "bf16"))
    np.testing.assert_array_equal(tp_keys, run_keys)


@pytest.mark.parametrize("budget", [52, 17])
def test_sm_budget_same_result(cuda_lib, budget):
    """A refresh confined to an SM budget (persistent clusters looping over
    more (query tile, label part) units) returns exactly the same keys."""
    from paper_2409_20156_b200 import _lib

    rng = np.random.default_rng(budget)
    L, d, nq, k = 70_000, 128, 1500, 48
    W = rng.uniform(-1 / np.sqrt(d), 1 / np.sqrt(d), size=(L, d)).astype(np.float32)
    E = rng.standard_normal((nq, d)).astype(np.float32)
    positives = random_positives(rng, nq, L, 0, 6)
    for flag in ("0", "1"):
        full_keys, _, _ = _with_two_pass(flag, lambda: _run(E, W, positives, k, "bf16"))
        _lib.set_refresh_sm_budget(budget)
        try:
            b_keys, _, _ = _with_two_pass(flag, lambda: _run(E, W, positives, k, "bf16"))
        finally:
            _lib.set_refresh_sm_budget(0)
        np.testing.assert_array_equal(b_keys, full_keys)


def test_query_topk_batch_reuses_the_mips_kernel(cuda_lib):
    """anns.query_topk / query_topk_batch (anns.py:211-230, the UpToDateHard and
    evaluation path): fp32-exact ids equal the C oracle bit for bit, and the
    float64 ranking of the reference on well-separated scores."""
    from paper_2409_20156_b200 import anns

    rng = np.random.default_rng(11)
    L, d, N, k = 5000, 64, 37, 10
    W = rng.standard_normal((L, d)).astype(np.float32)
    Q = rng.standard_normal((N, d)).astype(np.float32)
    index = anns.build_exact(W)
    ids, scores = anns.query_topk_batch(index, Q, k)
    _, oids, oscores = co.refresh_fp32(Q, W, np.zeros(N + 1, np.int64), np.zeros(0, np.int32), k)
    np.testing.assert_array_equal(ids, oids)
    np.testing.assert_array_equal(scores, oscores.astype(np.float64))
    s64 = W.astype(np.float64) @ Q.astype(np.float64).T
    for i in range(N):
        order = np.lexsort((np.arange(L), -s64[:, i]))[:k]
        assert ids[i].tolist() == order.tolist()
    one = anns.query_topk(index, Q[3], k)
    assert one.label_ids.tolist() == ids[3].tolist()


@pytest.mark.parametrize("k", [16, 64])
def test_bf16_rerank_from_bf16_labels(cuda_lib, k):
    """bf16 W (no fp32 copy): BF16_RERANK re-scores the bf16 rows exactly, so
    the ids equal FP32_EXACT run on the bf16-rounded W."""
    from paper_2409_20156_b200 import ops

    rng = np.random.default_rng(k)
    L, d, nq = 30_000, 256, 300
    W = rng.uniform(-1 / np.sqrt(d), 1 / np.sqrt(d), size=(L, d)).astype(np.float32)
    E = rng.standard_normal((nq, d)).astype(np.float32)
    positives = random_positives(rng, nq, L, 0, 5)
    Wb = ops.f32_to_bf16(dev(W))
    W_rounded = Wb.float().cpu().numpy()
    ip, pid = csr(positives)
    keys, ids, scores = ops.refresh_topk(dev(E), dev(ip), dev(pid), k, "bf16_rerank", labels_bf16=Wb)
    _, exact_ids, exact_scores = _run(E, W_rounded, positives, k, "fp32")
    np.testing.assert_array_equal(ids.cpu().numpy(), exact_ids)
    np.testing.assert_array_equal(scores.cpu().numpy(), exact_scores)


@pytest.mark.parametrize("n", [1, 3, 4, 1023, 4096 * 37 + 5, 7_077_888])
def test_f32_to_bf16_matches_torch_rne(cuda_lib, n):
    """The snapshot conversion is round-to-nearest-even, like torch's cast,
    for every length (vector body + tails)."""
    from paper_2409_20156_b200 import ops

    x = torch.randn(n, device="cuda") * 3
    x[: min(n, 4)] = torch.tensor([0.0, -0.0, 1e-40, 3.0e38][: min(n, 4)], device="cuda")
    got = ops.f32_to_bf16(x)
    assert torch.equal(got.view(torch.int16), x.to(torch.bfloat16).view(torch.int16))


@pytest.mark.parametrize("nq,L,d,k,offset", [(256, 20000, 128, 32, 0), (300, 9000, 768, 64, 0), (1, 5000, 256, 8, 0),
                                             (130, 1037, 128, 16, 5000), (512, 60000, 768, 200, 0)])
def test_fp8_rerank_equals_fp32(cuda_lib, nq, L, d, k, offset):
    """e4m3 candidate pass (tcgen05 kind::f8f6f4) + fp32 re-rank: ids equal
    the fp32-exact ones (the north star's >= 0.999 recall, here exact)."""
    rng = np.random.default_rng(nq + d)
    W = rng.uniform(-1 / np.sqrt(d), 1 / np.sqrt(d), size=(L, d)).astype(np.float32)
    E = rng.standard_normal((nq, d)).astype(np.float32)
    positives = [p + offset for p in random_positives(rng, nq, L, 0, 5)]
    _, exact_ids, exact_scores = _run(E, W, positives, k, "fp32", offset=offset)
    _, f8_ids, f8_scores = _run(E, W, positives, k, "fp8_rerank", offset=offset)
    recall = np.mean([len(set(a) & set(b)) / k for a, b in zip(f8_ids.tolist(), exact_ids.tolist())])
    assert recall >= 0.999, recall
    np.testing.assert_array_equal(f8_ids, exact_ids)
    np.testing.assert_array_equal(f8_scores, exact_scores)  # re-ranked scores are the fp32-exact ones


def test_quantize_e4m3_matches_torch(cuda_lib):
    """astra_quantize_e4m3 = torch's float8_e4m3fn cast of x * 448 / max|x| (RNE)."""
    import torch

    from paper_2409_20156_b200 import ops

    rng = np.random.default_rng(2)
    x = torch.from_numpy((rng.standard_normal(4096 * 3) * 0.05).astype(np.float32)).cuda()
    q = ops.quantize_e4m3(x)
    ref = (x * (448.0 / x.abs().max())).to(torch.float8_e4m3fn).view(torch.uint8)
    assert torch.equal(q, ref)
    xb = x.to(torch.bfloat16)
    qb = ops.quantize_e4m3(xb)
    refb = (xb.float() * (448.0 / xb.float().abs().max())).to(torch.float8_e4m3fn).view(torch.uint8)
    assert torch.equal(qb, refb)


def test_rerank_candidates_matches_oracle(cuda_lib):
    """astra_rerank_candidates (the sharded refresh's fp32 re-rank): all of the
    bf16 top-k' kept -> the BF16_RERANK result; a filtered candidate set (keys
    below a per-row threshold zeroed, as engine._refresh_sharded_rerank does)
    -> the fp32-exact top-k of that subset, key for key vs the C oracle."""
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import oracle_backend
    from paper_2409_20156_b200 import ops

    rng = np.random.default_rng(11)
    L, d, nq, k, off = 30_000, 256, 96, 24, 5000
    W = rng.uniform(-0.1, 0.1, size=(L, d)).astype(np.float32)
    E = rng.standard_normal((nq, d)).astype(np.float32)
    pos = [np.sort(rng.choice(L, size=3, replace=False)) + off for _ in range(nq)]
    ip = np.zeros(nq + 1, np.int64)
    ip[1:] = np.cumsum([len(p) for p in pos])
    pid = np.concatenate(pos).astype(np.int32)
    Wd, Ed = torch.from_numpy(W).cuda(), torch.from_numpy(E).cuda()
    ipd, pidd = torch.from_numpy(ip).cuda(), torch.from_numpy(pid).cuda()
    kc = ops.rerank_candidates_count(k)
    ck, _, _ = ops.refresh_topk(Ed, ipd, pidd, kc, "bf16", labels_f32=Wd, labels_bf16=ops.f32_to_bf16(Wd),
                                label_offset=off)
    full, _, _ = ops.rerank_candidates(Ed, ck, k, labels_f32=Wd, label_offset=off)
    ref, _, _ = ops.refresh_topk(Ed, ipd, pidd, k, "bf16_rerank", labels_f32=Wd, labels_bf16=ops.f32_to_bf16(Wd),
                                 label_offset=off)
    np.testing.assert_array_equal(full.cpu().numpy(), ref.cpu().numpy())
    cut = rng.integers(1, kc, size=nq)  # keep a prefix of random length per row
    mask = torch.arange(kc, device="cuda")[None, :] < torch.from_numpy(cut).cuda()[:, None]
    sub = torch.where(mask, ck, torch.zeros_like(ck))
    got, ids, _ = ops.rerank_candidates(Ed, sub, k, labels_f32=Wd, label_offset=off)
    want, want_ids, _ = oracle_backend.rerank_candidates(torch.from_numpy(E), sub.cpu(), k,
                                                         labels_f32=torch.from_numpy(W), label_offset=off)
    np.testing.assert_array_equal(got.cpu().numpy(), want.numpy())
    np.testing.assert_array_equal(ids.cpu().numpy(), want_ids.numpy())


@pytest.mark.parametrize("n_shards,global_candidates", [(2, False), (3, False), (2, True), (3, True)])
def test_sharded_rerank_composition_equals_one_gpu(cuda_lib, n_shards, global_candidates):
    """engine._refresh_sharded_rerank's composition on CUDA with the label
    range split into shards on one device: each shard's bf16 top-k', the
    owner's merge -> the global k'-th key tau, each shard's fp32 re-rank of
    its candidates >= tau, the merge of the fp32 lists — equals the one-GPU
    BF16_RERANK result key for key (the candidate set is the same)."""
    from paper_2409_20156_b200 import ops
    from paper_2409_20156_b200.shard import shard_range

    rng = np.random.default_rng(5)
    L, d, nq, k = 600_000, 256, 512, 48
    W = torch.from_numpy((rng.standard_normal((L, d)) / 16).astype(np.float32)).cuda()
    Wb = ops.f32_to_bf16(W)
    E = torch.from_numpy(rng.standard_normal((nq, d)).astype(np.float32)).cuda()
    pos = [np.sort(rng.choice(L, size=4, replace=False)).astype(np.int32) for _ in range(nq)]
    ip = torch.from_numpy(np.concatenate([[0], np.cumsum([len(p) for p in pos])]).astype(np.int64)).cuda()
    pid = torch.from_numpy(np.concatenate(pos)).cuda()
    want, want_ids, _ = ops.refresh_topk(E, ip, pid, k, "bf16_rerank", labels_f32=W, labels_bf16=Wb)
    kc = ops.rerank_candidates_count(k)
    ranges = [shard_range(L, r, n_shards) for r in range(n_shards)]
    if global_candidates:
        # engine._candidates_global: the shards' sample statistics -> the global
        # j-th largest group maximum -> local candidates at or above it -> the
        # summed counts / overflow flags -> the verify pass on every shard
        j = ops.refresh_plan_j(nq, min(hi - lo for lo, hi in ranges), d, kc)
        assert j > 0
        tops = [ops.refresh_sharded_stage(1, E, ip, pid, kc, Wb[lo:hi].contiguous(), label_offset=lo)
                for lo, hi in ranges]
        allv = torch.cat([t.to(torch.int64) & 0xFFFFFFFF for t in tops], dim=1)
        tau = allv.topk(j, dim=1).values[:, j - 1] << 32
        st2 = [ops.refresh_sharded_stage(2, E, ip, pid, kc, Wb[lo:hi].contiguous(), label_offset=lo, tau_keys=tau)
               for lo, hi in ranges]
        cnt = sum(c.to(torch.int64) for _, c, _ in st2)
        ovf = torch.stack([f for _, _, f in st2]).amax(0)
        need = ((cnt < kc) | (ovf > 0)).to(torch.int32)
        ck = [ops.refresh_sharded_stage(3, E, ip, pid, kc, Wb[lo:hi].contiguous(), label_offset=lo, io_keys=keys,
                                        flags=need) for (lo, hi), (keys, _, _) in zip(ranges, st2)]
        print(f"[sharded global candidates] {int(need.sum())} of {nq} queries verified")
    else:
        ck = [ops.refresh_topk(E, ip, pid, kc, "bf16", labels_f32=W[lo:hi].contiguous(),
                               labels_bf16=Wb[lo:hi].contiguous(), label_offset=lo)[0] for lo, hi in ranges]
    merged, _, _ = ops.topk_merge(torch.stack(ck), kc)
    tau = merged[:, kc - 1]
    flip = torch.tensor(-(2 ** 63), dtype=torch.int64, device="cuda")
    fk = []
    kept = 0
    for (lo, hi), c in zip(ranges, ck):
        keep = (c ^ flip) >= (tau[:, None] ^ flip)
        kept += int(keep.sum())
        cand = torch.where(keep, c, torch.zeros_like(c))
        fk.append(ops.rerank_candidates(E, cand, k, labels_f32=W[lo:hi].contiguous(), label_offset=lo)[0])
    got, got_ids, _ = ops.topk_merge(torch.stack(fk), k)
    assert kept == nq * kc  # exactly the global top-k' (keys are unique)
    np.testing.assert_array_equal(got.cpu().numpy(), want.cpu().numpy())
    np.testing.assert_array_equal(got_ids.cpu().numpy(), want_ids.cpu().numpy())
