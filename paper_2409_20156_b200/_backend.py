"""The device-op backend used by the reference-facing mirror (anns / trainer /
classifiers). The product backend is the CUDA C-ABI (`ops`); only tests swap
in another object with the same functions, explicitly, via install(backend=...)
or set_backend(). There is no automatic fallback."""

from __future__ import annotations

_active = None


def get():
    global _active
    if _active is None:
        from . import ops

        _active = ops
    return _active


def set_backend(backend) -> None:
    global _active
    _active = backend


def device():
    """Device the active backend computes on."""
    import torch

    dev = getattr(get(), "DEVICE", None)
    return torch.device(dev) if dev is not None else torch.device("cuda")
