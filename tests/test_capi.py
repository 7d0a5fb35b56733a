"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads without
a GPU, exports every symbol the header declares, and carries tcgen05/TMA SASS."""

import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "astra_b200.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(astra_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2409_20156_b200 import _lib, build

    build.build()
    lib = _lib.load()
    declared = _declared()
    assert declared, "header parse failed"
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.EXPORTED)
    assert b"sm_100a" in lib.astra_version()


def test_sass_has_tcgen05_and_tma():
    from paper_2409_20156_b200 import build

    lib = build.build()
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    if not sass:
        pytest.skip("cuobjdump unavailable")
    assert "UTCHMMA" in sass  # tcgen05.mma
    assert "UTMALDG" in sass  # TMA tensor loads
    assert "LDTM" in sass  # tcgen05.ld


def test_status_codes_map_to_reference_errors():
    from paper_2409_20156_b200.errors import ConfigError, DataError, NumericalError, raise_for_status

    for code, cls in ((2, ConfigError), (3, DataError), (4, NumericalError)):
        with pytest.raises(cls):
            raise_for_status(code, "x")
