"""The drop-in trainer's device mirror of a ClassifierBank (trainer.DeviceBank):
host-side row updates through classifiers.apply_classifier_updates_arrays keep
the mirror and its max|W| bound (which gates the single-pass step) in step
with the host array. CPU: oracle backend (host logic)."""

from dataclasses import dataclass

import numpy as np
import pytest

import oracle_backend
from paper_2409_20156_b200 import _backend, classifiers
from paper_2409_20156_b200.trainer import DeviceBank


@dataclass
class _Bank:
    weights: np.ndarray


class _Owner:
    pass


@pytest.fixture
def oracle():
    prev = _backend.get()
    _backend.set_backend(oracle_backend)
    yield
    _backend.set_backend(prev)


def test_mirror_follows_host_row_updates(oracle):
    rng = np.random.default_rng(0)
    bank = _Bank(rng.uniform(-0.1, 0.1, (50, 8)).astype(np.float32))
    owner = _Owner()
    db = DeviceBank.for_bank(owner, bank)
    assert DeviceBank.for_bank(owner, bank) is db
    assert float(db.w_absmax.item()) == pytest.approx(float(np.abs(bank.weights).max()))
    ids = np.array([3, 7, 11], dtype=np.int64)
    grads = rng.standard_normal((3, 8)).astype(np.float32) * 50
    classifiers.apply_classifier_updates_arrays(bank, ids, grads, 0.5, 0.0)
    np.testing.assert_array_equal(db.W.numpy(), bank.weights)  # mirror == host, bit for bit
    assert float(db.w_absmax.item()) >= float(np.abs(bank.weights).max())  # the bound still holds


def test_new_array_gets_a_new_mirror(oracle):
    bank = _Bank(np.ones((4, 2), np.float32))
    owner = _Owner()
    db = DeviceBank.for_bank(owner, bank)
    bank.weights = np.zeros((4, 2), np.float32)
    db2 = DeviceBank.for_bank(owner, bank)
    assert db2 is not db and float(db2.w_absmax.item()) == 0.0
    DeviceBank.update_rows(_Bank(np.ones((1, 2), np.float32)), [0], db.W[:1])  # no mirror: no-op


@pytest.mark.gpu
def test_mirror_step_and_host_updates_cuda(cuda_lib):
    """The drop-in's CUDA flow: a step on the mirror with its bound (the single
    pass), write-back of the touched rows, then a host-side row update — mirror,
    host and bound stay consistent and match the oracle."""
    import torch

    from oracle import xcmix_port as port
    from paper_2409_20156_b200 import ops

    rng = np.random.default_rng(4)
    L, d, B, S = 3000, 128, 32, 60
    W = rng.uniform(-1 / np.sqrt(d), 1 / np.sqrt(d), (L, d)).astype(np.float32)
    bank = _Bank(W.copy())
    db = DeviceBank.for_bank(_Owner(), bank)
    emb = rng.standard_normal((B, d)).astype(np.float32)
    ids = rng.integers(0, L, (B, S)).astype(np.int64)
    y = (rng.random((B, S)) < 0.05).astype(np.int8)
    origin = np.full(S, port.ORIGIN_RAND, np.int8)
    origin[:2] = port.ORIGIN_POS
    weights = np.full(S, 40.0, np.float32)
    weights[:2] = 1.0
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    ids_d = cu(ids.astype(np.int32))
    res = ops.slate_step(cu(emb), ids_d, cu(y), cu(origin), cu(weights), db.W, 0.1, 1e-4, w_absmax=db.w_absmax)
    db.sync_rows(torch.unique(ids_d))
    Wref = W.copy()
    loss, _, _, uids = port.slate_step(Wref, emb, None, ids, y, origin, weights, 0.1, 1e-4)
    assert res.status_host() == [0, 0, 0, 0]
    assert abs(res.loss - loss) <= 1e-5 * abs(loss)
    np.testing.assert_allclose(bank.weights[uids], Wref[uids], rtol=1e-5, atol=1e-6 * np.abs(Wref).max())
    np.testing.assert_array_equal(db.W.cpu().numpy(), bank.weights)
    grads = rng.standard_normal((4, d)).astype(np.float32) * 100
    classifiers.apply_classifier_updates_arrays(bank, np.array([0, 5, 9, 13]), grads, 0.5)
    np.testing.assert_array_equal(db.W.cpu().numpy(), bank.weights)
    assert float(db.w_absmax.item()) >= float(np.abs(bank.weights).max())
