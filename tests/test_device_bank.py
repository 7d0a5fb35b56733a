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
    db = DeviceBank.attach(bank)
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
    db.mark_updated()  # the device copy is now newer: the next host read copies it back
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


def test_lazy_host_sync_and_device_row_updates(oracle):
    """The device copy is authoritative while the drop-in trains: host reads
    of bank.weights copy it back (in place: aliases stay valid), shape queries
    do not, row updates through apply_classifier_updates_arrays run on the
    device copy, and assigning a new array drops the mirror."""
    import torch

    from paper_2409_20156_b200.bank import DeviceBank as DB

    @dataclass
    class Bank:
        weights: np.ndarray

        @property
        def n_labels(self):
            return self.weights.shape[0]

    host = np.zeros((6, 3), np.float32)
    bank = Bank(host)
    m = DB.attach(bank)
    assert DB.attach(bank) is m and isinstance(bank, Bank)
    m.W += 1.0  # a "step" on the device copy
    m.mark_updated()
    assert host.sum() == 0.0  # nothing copied yet
    assert bank.n_labels == 6 and m.dirty  # shape queries do not sync
    w = bank.weights
    assert w is host and host.sum() == 18.0 and not m.dirty
    classifiers.apply_classifier_updates_arrays(bank, np.array([1, 4]), np.ones((2, 3), np.float32), 0.5, 0.0)
    assert m.dirty and host[1, 0] == 1.0  # updated on the device only
    np.testing.assert_array_equal(bank.weights[[1, 4]], np.full((2, 3), 0.5, np.float32))
    assert float(m.w_absmax.item()) >= 0.5  # the bound covers the updated rows
    bank.weights = np.full((6, 3), 7.0, np.float32)
    assert DB.of(bank) is None
    m2 = DB.attach(bank)
    assert m2 is not m and float(m2.W[0, 0]) == 7.0
    host2 = bank.weights
    host2[2] = -3.0  # a direct in-place host write must be announced
    DB.host_modified(bank)
    assert float(m2.W[2, 0]) == -3.0 and not torch.equal(m2.W[2], m2.W[0])
