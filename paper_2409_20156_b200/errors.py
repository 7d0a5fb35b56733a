"""Error classes of the drop-in boundary.

The reference maps ConfigError/DataError/NumericalError to CLI exit codes
2/3/4 (errors.py:1-21, cli.py:91-105); the C-ABI returns the same codes.
When the reference package is importable (we are running under it as a
drop-in) its own classes are reused, so `except xcmix.errors.ConfigError`
in the caller catches errors raised here.
"""

try:  # pragma: no cover - depends on the caller's environment
    from xcmix.errors import ConfigError, DataError, NumericalError, XcmixError
except ImportError:  # standalone (e.g. the GPU box has no reference tree)

    class XcmixError(Exception):
        pass

    class ConfigError(XcmixError):
        """Bad run configuration (exit code 2)."""

    class DataError(XcmixError):
        """Malformed data or out-of-range ids (exit code 3)."""

    class NumericalError(XcmixError):
        """Non-finite values where finite ones are required (exit code 4)."""


class CudaError(RuntimeError):
    """A CUDA runtime failure inside the library (status 5)."""


_BY_CODE = {2: ConfigError, 3: DataError, 4: NumericalError, 5: CudaError}


def raise_for_status(code: int, message: str) -> None:
    if code:
        raise _BY_CODE.get(code, CudaError)(message or f"astra status {code}")
