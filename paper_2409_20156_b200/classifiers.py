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
    W = bank.weights
    rows = torch.from_numpy(np.ascontiguousarray(W[ids], dtype=np.float32)).to(dev)
    g = torch.from_numpy(np.ascontiguousarray(grads, dtype=np.float32).reshape(len(ids), -1)).to(dev)
    local = torch.arange(len(ids), dtype=torch.int64, device=dev)
    ops.apply_updates(rows, local, g, float(lr), float(weight_decay))  # raises before writing
    W[ids] = rows.cpu().numpy()
    # keep the trainer's device mirror of this bank (if any) and its max|W|
    # bound in step with the host array
    from .trainer import DeviceBank

    DeviceBank.update_rows(bank, ids, rows)
