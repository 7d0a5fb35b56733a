"""A whole reference `train()` run through the drop-in, against a golden
recorded from the unmodified reference (tests/golden/make_golden.py, fixture
train_run.npz: planted synthetic data, 4 epochs, Mixture strategy, tau_s=2,
tau_r=1 — the refresh pipeline snapshots at the end of epoch c-2 and the
cache is consumed from epoch 2 on — embed_dim=128, eval every 2 epochs).

install(slates="reference") keeps the reference's PCG64 slates, so the drop-in
run sees the same slate indices; everything on the hot path (shortlist
refresh, sampled loss/gradients, W update, dense probe, P@k) runs on the
selected backend: the CUDA library on the GPU, the oracle stand-in on CPU.
Per-epoch losses and probe within 1e-5 relative, P@k equal, final W and the
encoder's projection within 1e-5 relative + 1e-6 * max|.| absolute.
"""

import os
import sys

import numpy as np
import pytest

from conftest import ROOT, golden

REF_PKG = os.path.join(ROOT, "baseline", "_ref")
REF_SRC = "/root/reference/pkg/src"


def _reference_path():
    for p in (REF_PKG, REF_SRC):
        if os.path.isdir(os.path.join(p, "xcmix")):
            return p
    return None


def _inputs():
    import xcmix.dataset as xd
    import xcmix.trainer as xt

    from golden_train_spec import TRAIN_CONFIG, TRAIN_SPEC

    sp_ = TRAIN_SPEC
    train, ev = xd.generate_synthetic(sp_["n_points"], sp_["n_features"], sp_["n_labels"], sp_["labels_per_point"],
                                      noise_level=sp_["noise_level"], seed=sp_["seed"])
    return train, ev, xt.TrainConfig(**TRAIN_CONFIG)


def _train_through_dropin(backend):
    path = _reference_path()
    if path is None:
        pytest.skip("reference package not available (baseline/_ref)")
    for p in (path, os.path.join(ROOT, "tests", "golden")):
        if p not in sys.path:
            sys.path.insert(0, p)
    import xcmix.anns as xa
    import xcmix.trainer as xt

    from paper_2409_20156_b200 import install as inst

    inst.install(backend=backend, slates="reference")
    try:
        train, ev, cfg = _inputs()
        enc, bank, log = xt.train(train, cfg, eval_dataset=ev)
        consume = [e["epoch"] for e in log.events if e["stage"] == xa.STAGE_CONSUME]
        return enc, bank, log, consume
    finally:
        inst.uninstall()


def _compare(enc, bank, log, consume):
    g = golden("train_run.npz")
    rec = log.records
    loss = np.array([r.mean_slate_loss for r in rec])
    probe = np.array([r.probe_full_loss for r in rec])
    print("loss", loss, "golden", g["loss"])
    np.testing.assert_allclose(loss, g["loss"], rtol=1e-5)
    np.testing.assert_allclose(probe, g["probe"], rtol=1e-5)
    p1 = np.array([np.nan if r.p_at_1 is None else r.p_at_1 for r in rec])
    p5 = np.array([np.nan if r.p_at_5 is None else r.p_at_5 for r in rec])
    np.testing.assert_array_equal(p1, g["p1"])
    np.testing.assert_array_equal(p5, g["p5"])
    np.testing.assert_array_equal([r.snapshot_epoch for r in rec], g["snapshot"])
    np.testing.assert_array_equal(consume, g["consume"])
    W = bank.weights
    np.testing.assert_allclose(W, g["W"], rtol=1e-5, atol=1e-6 * np.abs(g["W"]).max())
    np.testing.assert_allclose(enc.projection, g["projection"], rtol=1e-5, atol=1e-6 * np.abs(g["projection"]).max())


def test_train_golden_oracle_backend():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_backend

    _compare(*_train_through_dropin(oracle_backend))


@pytest.mark.gpu
def test_train_golden_cuda(cuda_lib):
    from paper_2409_20156_b200 import _lib

    n0 = _lib.launch_count()
    out = _train_through_dropin(None)
    assert _lib.launch_count() - n0 > 100  # the run went through libastra_b200
    _compare(*out)
