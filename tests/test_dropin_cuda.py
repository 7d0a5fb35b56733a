"""The reference's OWN test-suite through the drop-in on CUDA.

`install()` rebinds xcmix's hot-path functions (retrieve_hard_negatives,
build_exact / query_topk / predict_topk, _assemble_batch_slates,
_batch_forward_backward, apply_classifier_updates_arrays, the dense probes and
the full-loss arm) to the B200 path with the CUDA backend (libastra_b200), and
the reference's tests — unit suites plus the acceptance criteria
(test_acceptance.py: estimator unbiasedness, refresh pipeline stall,
bitwise determinism, ...) — run unchanged against it. The reference package
and its tests come from baseline/_ref / baseline/_ref_tests, which
__graft_entry__.build() installs from /root/reference and which travel to the
GPU box with the snapshot (the reference tree itself does not).
"""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

REF_PKG = os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(ROOT, "baseline", "_ref_tests")
SUITES = ["test_anns.py", "test_classifiers.py", "test_sampler.py", "test_loss.py", "test_trainer.py",
          "test_encoder.py", "test_eval.py", "test_acceptance.py"]


def _run(slates, suites=SUITES, extra=()):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF_PKG, ROOT, os.path.join(ROOT, "tests")])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    env["ASTRA_DROPIN_SLATES"] = slates
    env["ASTRA_DROPIN_BACKEND"] = "cuda"
    cmd = [sys.executable, "-m", "pytest", *[os.path.join(REF_TESTS, s) for s in suites], "-p", "dropin_plugin",
           "-p", "no:cacheprovider", "-q", "-rf", *extra]
    return subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=1800, cwd=REF_TESTS)


@pytest.mark.skipif(not os.path.isdir(REF_TESTS) or not os.path.isdir(os.path.join(REF_PKG, "xcmix")),
                    reason="baseline/_ref(_tests) not installed (run __graft_entry__.build() where /root/reference exists)")
@pytest.mark.parametrize("slates", ["philox", "reference"])
def test_reference_suite_on_cuda(cuda_lib, slates):
    r = _run(slates)
    out = r.stdout + r.stderr
    print(out[-4000:])
    assert r.returncode == 0, out[-4000:]
    assert " passed" in r.stdout
    # the CUDA library, not a fallback, served the calls
    import re

    m = re.search(r"\[astra\] libastra_b200 kernel launches: (\d+)", out)
    assert m and int(m.group(1)) > 1000, "the drop-in did not run on libastra_b200"
