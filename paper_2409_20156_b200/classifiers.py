"""Drop-in for xcmix.classifiers.apply_classifier_updates_arrays
(classifiers.py:75-82): w <- w - lr*(g + wd*w) on unique touched rows, each
op rounded in fp32 like NumPy; NumericalError (nothing written) if any
gradient is non-finite. The arithmetic runs on the GPU (astra_apply_updates)."""

from __future__ import annotations

import numpy as np
import torch

from . import _backend
from .errors import NumericalError


def apply_classifier_updates_arrays(bank, ids, grads, lr, weight_decay=0.0) -> None:
    """Array form of apply_classifier_updates; ids must be unique."""
    ids = np.asarray(ids, dtype=np.int64)
    grads = np.asarray(grads)
    if grads.size and not np.issubdtype(grads.dtype, np.floating):
        grads = grads.astype(np.float32)
    if ids.size == 0:
        if grads.size and not np.isfinite(grads).all():
            raise NumericalError("non-finite classifier gradient")
        return
    ops = _backend.get()
    dev = _backend.device()
    from .bank import DeviceBank

    mirror = DeviceBank.of(bank)
    if mirror is not None:  # the drop-in trains this bank on the device: update there
        idx = torch.from_numpy(ids).to(mirror.W.device)
        rows = mirror.W[idx]
        g = torch.from_numpy(np.ascontiguousarray(grads, dtype=np.float32).reshape(len(ids), -1)).to(mirror.W.device)
        local = torch.arange(len(ids), dtype=torch.int64, device=mirror.W.device)
        ops.apply_updates(rows, local, g, float(lr), float(weight_decay))  # raises before writing
        mirror.W[idx] = rows
        if rows.numel():
            torch.maximum(mirror.w_absmax, rows.abs().amax().reshape(1).float(), out=mirror.w_absmax)
        mirror.mark_updated()
        return
    W = bank.weights
    rows = torch.from_numpy(np.ascontiguousarray(W[ids], dtype=np.float32)).to(dev)
    g = torch.from_numpy(np.ascontiguousarray(grads, dtype=np.float32).reshape(len(ids), -1)).to(dev)
    local = torch.arange(len(ids), dtype=torch.int64, device=dev)
    ops.apply_updates(rows, local, g, float(lr), float(weight_decay))  # raises before writing
    W[ids] = rows.cpu().numpy()
