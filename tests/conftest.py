"""Shared pytest setup: the `gpu` marker and import paths.

`-m "not gpu"` tests run in the build container (no GPU): oracle vs golden
fixtures, host logic, C-ABI symbol exports, gloo multi-process logic.
`-m gpu` tests run on a B200 through the C-ABI library and compare with the
oracle (tests/ is the only place allowed to import oracle/).
"""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def golden(name):
    import numpy as np

    return dict(np.load(os.path.join(GOLDEN, name), allow_pickle=False))


@pytest.fixture
def cuda_lib():
    """The CUDA C-ABI library; GPU tests fail loudly if it cannot be loaded."""
    import torch

    assert torch.cuda.is_available(), "gpu test without a CUDA device"
    from paper_2409_20156_b200 import _lib

    return _lib.load()
