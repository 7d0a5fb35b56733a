"""pytest plugin (test infrastructure): install the B200 drop-in into the
reference package BEFORE the reference's own test modules are imported, so
`from xcmix.anns import retrieve_hard_negatives` etc. bind to the mirror.

ASTRA_DROPIN_BACKEND=oracle (default) runs the device ops on the CPU oracle
(host-logic check, build container); =cuda uses libastra_b200 on a GPU.
ASTRA_DROPIN_SLATES=philox|reference chooses the slate sampler.
"""

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (ROOT, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    from paper_2409_20156_b200.install import install

    backend = None
    if os.environ.get("ASTRA_DROPIN_BACKEND", "oracle") == "oracle":
        import oracle_backend

        backend = oracle_backend
    install(backend=backend, slates=os.environ.get("ASTRA_DROPIN_SLATES", "philox"))


def pytest_terminal_summary(terminalreporter):
    """With the CUDA backend: report how many kernels libastra_b200 launched
    (tests/test_dropin_cuda.py checks it is > 0: no silent host fallback)."""
    if os.environ.get("ASTRA_DROPIN_BACKEND", "oracle") != "cuda":
        return
    from paper_2409_20156_b200 import _lib

    terminalreporter.write_line(f"[astra] libastra_b200 kernel launches: {_lib.launch_count()}")
