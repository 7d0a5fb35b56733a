"""Device-resident classifier weights behind the reference's ClassifierBank.

The reference keeps W as the numpy array `bank.weights` (classifiers.py:13-24)
and reads it on the host at a few boundaries only: the refresh snapshot
(`_refresh_fn`, trainer.py:429-430), the per-epoch probes (`_probe_full_loss`,
`_eval_p_at`, trainer.py:398-423), `save_checkpoint` (:689-710), evaluation and
the caller after `train()` returns. Its only in-place writer is
`apply_classifier_updates_arrays` (classifiers.py:75-82), which the drop-in
rebinds.

`DeviceBank.attach(bank)` uploads W once and makes the device copy
authoritative: the sampled steps update it in place (no per-step write-back),
and the bank's class is swapped for a subclass whose `weights` property copies
the device W back to the host array (one D2H, in place, so the array object
and every alias of it stay valid) the first time host code reads it after a
device update. Assigning a new array to `bank.weights` drops the mirror (the
next attach uploads the new array). Host code that writes INTO the array
returned by `bank.weights` outside `apply_classifier_updates_arrays` must call
`DeviceBank.host_modified(bank)` afterwards.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _backend

_LAZY_CLASSES: dict[type, type] = {}


def _lazy_class(base: type) -> type:
    """Subclass of `base` whose `weights` reads sync from the device mirror."""
    cls = _LAZY_CLASSES.get(base)
    if cls is not None:
        return cls

    def _get(self):
        m = self.__dict__.get("_astra_mirror")
        if m is not None:
            m.sync_host()
        return self.__dict__["weights"]

    def _set(self, value):
        self.__dict__["weights"] = value
        self.__dict__.pop("_astra_mirror", None)  # a new array: re-uploaded on next attach

    ns = {"weights": property(_get, _set), "__module__": base.__module__, "__qualname__": base.__qualname__}
    # shape queries must not force a device->host copy
    if isinstance(getattr(base, "n_labels", None), property):
        ns["n_labels"] = property(lambda self: self.__dict__["weights"].shape[0])
    if isinstance(getattr(base, "dim", None), property):
        ns["dim"] = property(lambda self: self.__dict__["weights"].shape[1])
    cls = type(base.__name__, (base,), ns)
    _LAZY_CLASSES[base] = cls
    return cls


class DeviceBank:
    """fp32 device copy of a bank's weights plus its running max|W| bound."""

    def __init__(self, host: np.ndarray):
        self.host = host
        # (a copy even on a CPU backend, so host and device never alias)
        self.W = torch.from_numpy(np.ascontiguousarray(host, dtype=np.float32)).to(_backend.device(), copy=True)
        # running max|W| bound, kept current by every step: lets astra_slate_step
        # prove finiteness up front and take the single label-major pass
        self.w_absmax = (self.W.abs().amax().reshape(1).float() if self.W.numel()
                         else torch.zeros(1, dtype=torch.float32, device=self.W.device))
        self.dirty = False  # device newer than host

    # ------------------------------------------------------------ attach
    @classmethod
    def attach(cls, bank) -> "DeviceBank":
        host = bank.__dict__["weights"] if "weights" in bank.__dict__ else bank.weights
        m = bank.__dict__.get("_astra_mirror")
        if m is not None and m.host is host:
            return m
        m = cls(host)
        if not isinstance(type(bank).__dict__.get("weights"), property):
            try:
                bank.__class__ = _lazy_class(type(bank))
            except TypeError:  # e.g. __slots__: keep the host eagerly in step instead
                m.eager = True
        bank.__dict__["_astra_mirror"] = m
        return m

    @classmethod
    def for_bank(cls, owner, bank) -> "DeviceBank":  # round-1 name
        return cls.attach(bank)

    @staticmethod
    def of(bank) -> "DeviceBank | None":
        m = getattr(bank, "__dict__", {}).get("_astra_mirror")
        if m is not None and m.host is bank.__dict__.get("weights"):
            return m
        return None

    eager = False

    # ------------------------------------------------------------ sync
    def mark_updated(self) -> None:
        """The device W was updated (a step / row update ran on it)."""
        self.dirty = True
        if self.eager:
            self.sync_host()

    def sync_host(self) -> None:
        """Copy the device W into the host array, in place, if it is newer."""
        if not self.dirty:
            return
        if self.host.dtype == np.float32 and self.host.flags.c_contiguous and self.host.flags.writeable:
            torch.from_numpy(self.host).copy_(self.W)
        else:
            self.host[...] = self.W.cpu().numpy()
        self.dirty = False

    @staticmethod
    def host_modified(bank) -> None:
        """Host code wrote into bank.weights in place: re-upload it."""
        m = DeviceBank.of(bank)
        if m is None:
            return
        m.W.copy_(torch.from_numpy(np.ascontiguousarray(m.host, dtype=np.float32)))
        m.w_absmax.fill_(float(np.abs(m.host).max()) if m.host.size else 0.0)
        m.dirty = False

    @staticmethod
    def update_rows(bank, ids, rows_dev) -> None:
        """After a host-side row update of `bank`: copy the rows into the
        bank's device mirror, if one exists for this very array, and raise the
        max|W| bound to cover them."""
        m = DeviceBank.of(bank)
        if m is None:
            return
        idx = torch.as_tensor(np.asarray(ids, dtype=np.int64), device=m.W.device)
        r = rows_dev.to(m.W.device, m.W.dtype)
        m.W[idx] = r
        if r.numel():
            torch.maximum(m.w_absmax, r.abs().amax().reshape(1).float(), out=m.w_absmax)

    def sync_rows(self, ids: torch.Tensor) -> None:
        """Copy the given (device) rows back into the host array."""
        idx = ids.to(torch.int64)
        self.host[idx.cpu().numpy()] = self.W[idx].cpu().numpy()


def device_weights(bank) -> torch.Tensor:
    """The bank's current fp32 weights on the device: the live mirror when the
    drop-in trains this bank, else an upload of the host array (no caching:
    the host array may change in place)."""
    m = DeviceBank.of(bank)
    if m is not None:
        return m.W
    host = bank.__dict__["weights"] if "weights" in getattr(bank, "__dict__", {}) else bank.weights
    return torch.from_numpy(np.ascontiguousarray(host, dtype=np.float32)).to(_backend.device())
