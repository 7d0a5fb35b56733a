"""Run the REFERENCE's own test-suite through the drop-in (install()).

Only possible where the reference tree exists (the build container). The
device ops run on the CPU oracle backend here, so this checks the mirror's
host logic — signatures, dtypes, error classes, rebinding, write-back —
against the reference's 200+ tests; the kernels' parity is covered by the
-m gpu tests. With ASTRA_DROPIN_SLATES=reference the trainer path must be
bitwise the reference's (identical slates, the reference arithmetic)."""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

REF = "/root/reference/pkg"
SUITES = ["test_anns.py", "test_classifiers.py", "test_sampler.py", "test_loss.py", "test_trainer.py", "test_encoder.py",
          "test_eval.py"]


def _run(slates, extra=()):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(REF, "src"), ROOT, os.path.join(ROOT, "tests")])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    env["ASTRA_DROPIN_SLATES"] = slates
    env["ASTRA_DROPIN_BACKEND"] = "oracle"
    cmd = [sys.executable, "-m", "pytest", *[os.path.join(REF, "tests", s) for s in SUITES], "-p", "dropin_plugin",
           "-p", "no:cacheprovider", "-q", "-x", *extra]
    return subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree absent (GPU box)")
@pytest.mark.parametrize("slates", ["philox", "reference"])
def test_reference_suite_passes_through_dropin(slates):
    r = _run(slates)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    assert " passed" in r.stdout
