"""The all-negatives arm and the dense probes:
train_full_loss_baseline (trainer.py:563-616), _probe_full_loss (:398-403),
_eval_p_at (:406-423).

CPU (build container, reference importable): the drop-in mirror on the CPU
oracle backend reproduces the reference's own run bit for bit (same generator
stream, batch order, dropout, BLAS calls) — this pins the mirror's host logic
and the oracle restatement. The CUDA path is checked against the oracle in
test_gpu_full_loss.py."""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

REF = "/root/reference/pkg"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree absent (GPU box)")
def test_full_loss_arm_dropin_matches_reference_bitwise():
    code = f"""
import sys
ROOT, REF = {ROOT!r}, {REF!r}
sys.path[:0] = [ROOT, ROOT + "/tests", REF + "/src", REF + "/tests"]
import numpy as np
import oracle_backend
import xcmix.trainer as xt
from xcmix.dataset import generate_synthetic
from xcmix.trainer import TrainConfig
from paper_2409_20156_b200.install import install, uninstall

# the reference tests' tiny planted corpus and quick config (tests/conftest.py:9-11, test_trainer.py:27-34)
train_ds, test_ds = generate_synthetic(300, 64, 40, 2, noise_level=0.05, seed=11)
cfg = TrainConfig(epochs=3, batch_size=32, lr_encoder=0.02, lr_classifier=0.1, warmup_steps=4, k_r=8, k_h=4, k_p=2,
                  tau_s=3, tau_r=3, strategy="Mixture", eval_every=1, embed_dim=16, seed=0, dropout=0.1)
ref_enc, ref_bank, ref_log = xt.train_full_loss_baseline(train_ds, cfg, eval_dataset=test_ds)
install(backend=oracle_backend)
try:
    enc, bank, log = xt.train_full_loss_baseline(train_ds, cfg, eval_dataset=test_ds)
    assert xt.train_full_loss_baseline.__module__.startswith("paper_2409_20156_b200")
finally:
    uninstall()
np.testing.assert_array_equal(bank.weights, ref_bank.weights)
np.testing.assert_array_equal(enc.projection, ref_enc.projection)
assert len(log.records) == len(ref_log.records) == 3
for a, b in zip(log.records, ref_log.records):
    assert a.mean_slate_loss == b.mean_slate_loss, (a, b)
    assert abs(a.probe_full_loss - b.probe_full_loss) <= 1e-12 * abs(b.probe_full_loss), (a, b)
    assert (a.p_at_1, a.p_at_5) == (b.p_at_1, b.p_at_5), (a, b)
print("ok", len(log.records))
"""
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, (r.stdout + r.stderr)[-3000:]
