"""The synchronous-refresh snapshot ("snapshot without a full
W copy"): ClassifierEngine.snapshot(copy=False) aliases the live W, refreshes
from it equal the refreshes from a copied snapshot, and a refresh after W was
written raises ConfigError instead of reading weights newer than the snapshot.
CPU tests run the engine's host logic on the oracle backend; the gpu test
repeats it on the CUDA engine (fp32 W and bf16 W)."""

import numpy as np
import pytest
import torch

import oracle_backend
from paper_2409_20156_b200.engine import ClassifierEngine
from paper_2409_20156_b200.errors import ConfigError

L, D, K_P, K_H, K_R, B = 700, 128, 2, 6, 12, 24  # d % 128 == 0: the bf16 refresh and the single pass


def _inputs(device, seed=0):
    rng = np.random.default_rng(seed)
    emb = rng.standard_normal((B, D)).astype(np.float32)
    pos = [np.unique(rng.integers(0, L, 3)).astype(np.int32) for _ in range(B)]
    ip = np.zeros(B + 1, np.int64)
    ip[1:] = np.cumsum([len(p) for p in pos])
    t = (torch.from_numpy(emb), torch.from_numpy(ip), torch.from_numpy(np.concatenate(pos)),
         torch.arange(B, dtype=torch.int64))
    return tuple(x.to(device) for x in t)


def _check(device, backend, mode, w_dtype):
    W = np.random.default_rng(1).uniform(-0.1, 0.1, (L, D)).astype(np.float32)
    kw = dict(backend=backend) if backend is not None else {}
    eng = ClassifierEngine(L, D, k_p=K_P, k_h=K_H, k_r=K_R, weights=W, refresh_mode=mode, seed=5, device=device,
                           w_dtype=w_dtype, **kw)
    emb, ip, pid, rows = _inputs(device)
    eng.snapshot(0)
    ids_copy, sc_copy = eng.refresh(emb, ip, pid, K_H)
    eng.snapshot(0, copy=False)
    snap = eng.snap_bf16 if eng.snap_f32 is None else eng.snap_f32
    if w_dtype == torch.float32 or eng.snap_f32 is None:
        assert snap.data_ptr() == eng.W.data_ptr()  # aliased, no copy of W
    ids, sc = eng.refresh(emb, ip, pid, K_H)
    np.testing.assert_array_equal(ids.cpu().numpy(), ids_copy.cpu().numpy())
    np.testing.assert_array_equal(sc.cpu().numpy(), sc_copy.cpu().numpy())
    eng.refresh(emb, ip, pid, K_H)  # any number of refreshes before the next update
    sl = eng.sample(rows, ip, pid, ids, epoch=3, step=0)
    eng.step(emb, sl, 0.05, 1e-4)
    with pytest.raises(ConfigError):
        eng.refresh(emb, ip, pid, K_H)
    eng.snapshot(1)  # a copied snapshot is immune to later updates
    ids1, _ = eng.refresh(emb, ip, pid, K_H)
    eng.step(emb, eng.sample(rows, ip, pid, ids1, epoch=3, step=1), 0.05, 1e-4)
    ids2, _ = eng.refresh(emb, ip, pid, K_H)
    np.testing.assert_array_equal(ids1.cpu().numpy(), ids2.cpu().numpy())


@pytest.mark.parametrize("mode", ["fp32", "bf16_rerank"])
def test_aliased_snapshot_oracle_backend(mode):
    _check("cpu", oracle_backend, mode, torch.float32)


@pytest.mark.gpu
@pytest.mark.parametrize("mode,w_dtype", [("fp32", torch.float32), ("bf16_rerank", torch.float32),
                                          ("bf16_rerank", torch.bfloat16)])
def test_aliased_snapshot_cuda(mode, w_dtype):
    _check("cuda", None, mode, w_dtype)
