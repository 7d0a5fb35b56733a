"""Shard checkpoint of the GPU-resident state:
ClassifierEngine.save_shard / load_shard round-trip W (fp32 / bf16), the Adam
moments and step, and the max|W| bound exactly; a restored engine continues
bit-identically to one that never stopped. CPU tests run the engine on the
oracle backend (host logic); the gpu test repeats the round trip on the
device-resident CUDA engine."""

import numpy as np
import pytest
import torch

import oracle_backend
from paper_2409_20156_b200.engine import ClassifierEngine
from paper_2409_20156_b200.errors import ConfigError, DataError

L, D, K_P, K_H, K_R = 500, 32, 2, 4, 10


def _batch(rng, B=16):
    emb = rng.standard_normal((B, D)).astype(np.float32)
    pos = [np.unique(rng.integers(0, L, 3)).astype(np.int32) for _ in range(B)]
    ip = np.zeros(B + 1, np.int64)
    ip[1:] = np.cumsum([len(p) for p in pos])
    rows = np.arange(B, dtype=np.int64)
    return (torch.from_numpy(emb), torch.from_numpy(ip), torch.from_numpy(np.concatenate(pos)),
            torch.from_numpy(rows))


def _engine(device="cpu", backend=oracle_backend, optimizer="adam", w_dtype=torch.float32):
    W = np.random.default_rng(1).uniform(-0.1, 0.1, (L, D)).astype(np.float32)
    kw = dict(backend=backend) if backend is not None else {}
    return ClassifierEngine(L, D, k_p=K_P, k_h=K_H, k_r=K_R, weights=W, refresh_mode="fp32", seed=5, device=device,
                            optimizer=optimizer, w_dtype=w_dtype, **kw)


def _train(eng, steps, seed):
    rng = np.random.default_rng(seed)
    dev = eng.device
    for t in range(steps):
        emb, ip, pid, rows = (x.to(dev) for x in _batch(rng))
        eng.snapshot(t)
        ids, _ = eng.refresh(emb, ip, pid, K_H)
        sl = eng.sample(rows, ip, pid, ids, epoch=3, step=t)
        eng.step(emb, sl, 0.01, 1e-4)


def _roundtrip(tmp_path, device, backend, optimizer, w_dtype, train=True):
    a = _engine(device, backend, optimizer, w_dtype)
    if train:
        _train(a, 3, 0)
    else:  # (the oracle backend runs SGD only: stand-in optimizer state)
        g = torch.Generator().manual_seed(3)
        a.W.copy_(torch.rand(a.W.shape, generator=g).to(a.W.dtype))
        if optimizer == "adam":
            a.m.copy_(torch.randn(a.m.shape, generator=g))
            a.v.copy_(torch.rand(a.v.shape, generator=g))
            a.adam_step = 7
        a.w_absmax.fill_(1.5)
    path = str(tmp_path / "shard.xash")
    a.save_shard(path)
    b = _engine(device, backend, optimizer, w_dtype)
    b.load_shard(path)
    assert torch.equal(a.W.cpu().view(torch.int16) if w_dtype == torch.bfloat16 else a.W.cpu(),
                       b.W.cpu().view(torch.int16) if w_dtype == torch.bfloat16 else b.W.cpu())
    if optimizer == "adam":
        assert torch.equal(a.m.cpu(), b.m.cpu()) and torch.equal(a.v.cpu(), b.v.cpu())
    assert a.adam_step == b.adam_step and float(a.w_absmax.item()) == float(b.w_absmax.item())
    if train:
        _train(a, 2, 7)
        _train(b, 2, 7)
        assert torch.equal(a.W.float().cpu(), b.W.float().cpu())  # continues identically


def test_shard_checkpoint_roundtrip_cpu_sgd(tmp_path):
    _roundtrip(tmp_path, "cpu", oracle_backend, "sgd", torch.float32)


@pytest.mark.parametrize("w_dtype", [torch.float32, torch.bfloat16])
def test_shard_checkpoint_roundtrip_cpu_adam_state(tmp_path, w_dtype):
    _roundtrip(tmp_path, "cpu", oracle_backend, "adam", w_dtype, train=False)


def test_shard_checkpoint_rejects_mismatch(tmp_path):
    a = _engine()
    path = str(tmp_path / "s.xash")
    a.save_shard(path)
    with pytest.raises(ConfigError):
        _engine(optimizer="sgd").load_shard(path)
    with open(path, "r+b") as fh:
        fh.write(b"NOPE")
    with pytest.raises(DataError):
        _engine().load_shard(path)
    open(path, "wb").write(b"XA")
    with pytest.raises(DataError):
        _engine().load_shard(path)


@pytest.mark.gpu
@pytest.mark.parametrize("w_dtype", [torch.float32, torch.bfloat16])
def test_shard_checkpoint_roundtrip_gpu(tmp_path, cuda_lib, w_dtype):
    _roundtrip(tmp_path, "cuda", None, "adam", w_dtype)


def test_truncated_checkpoint_restores_nothing(tmp_path):
    """A truncated file raises DataError before anything is written: W, the
    bound and the snapshot of the target engine are left as they were."""
    a = _engine(optimizer="sgd")
    path = str(tmp_path / "t.xash")
    a.save_shard(path)
    data = open(path, "rb").read()
    open(path, "wb").write(data[:-100])
    b = _engine(optimizer="sgd")
    b.W.mul_(2.0)
    b.w_absmax.fill_(9.0)
    b.snapshot(0)
    before = b.W.clone()
    with pytest.raises(DataError):
        b.load_shard(path)
    assert torch.equal(b.W, before) and float(b.w_absmax.item()) == 9.0 and b.snap_f32 is not None
    open(path, "wb").write(data)
    b.load_shard(path)
    assert torch.equal(b.W, a.W) and b.snap_f32 is None  # the stale snapshot is dropped
