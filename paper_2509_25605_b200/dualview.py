"""DualView on real device memory — the B200 counterpart of the reference's
``LAPIS::DualView`` (runtime_header.py:93-236) and of the interpreter's
two-space SimBuffer (interp.py:90-123, 304-322).

A DualView is a pinned host tensor plus a device tensor sharing one record of
``modified_host`` / ``modified_device`` flags.  ``sync_device`` copies host ->
device only when the host side is modified (one H2D event of ``nbytes``);
``sync_host`` copies back only when the device side is modified.  Children
from ``subview`` alias the parent storage and share its flags.  Copies are
``cudaMemcpyAsync`` on the current stream (torch ``copy_(non_blocking=True)``
between pinned and device memory).  ``transfer_stats()`` counts exactly what
the reference's ``transferStats()`` counts (runtime_header.py:52-64), so the
counts can be compared with the interpreter's trace.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch


@dataclass
class TransferStats:
    h2d_count: int = 0
    d2h_count: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0


_STATS = TransferStats()


def transfer_stats() -> TransferStats:
    return _STATS


def reset_transfer_stats() -> None:
    global _STATS
    _STATS = TransferStats()


class _Record:
    __slots__ = ("host", "device", "modified_host", "modified_device", "label", "h2d_done")

    def __init__(self, host: torch.Tensor, device: torch.Tensor, label: str):
        self.host = host
        self.device = device
        self.modified_host = False
        self.modified_device = False
        self.label = label
        self.h2d_done = None   # event of an H2D copy that may still read the host side

    def host_quiescent(self) -> None:
        """Wait for an in-flight H2D copy out of the pinned host buffer: the
        reference's syncDevice is a blocking deep_copy, so the host side may be
        written as soon as it returns (runtime_header.py:145-160)."""
        if self.h2d_done is not None:
            self.h2d_done.synchronize()
            self.h2d_done = None


def _pinned_like(a, dtype=None) -> torch.Tensor:
    t = torch.as_tensor(np.ascontiguousarray(a)) if not isinstance(a, torch.Tensor) else a
    if dtype is not None:
        t = t.to(dtype)
    t = t.contiguous()
    try:
        return t.pin_memory()
    except RuntimeError:  # no CUDA driver: keep pageable memory (tests on CPU)
        return t.clone()


class DualView:
    """Mirrored host/device buffer with lazy coherence (see module docstring)."""

    def __init__(self, record: _Record, window: tuple[slice, ...] | None = None):
        self._rec = record
        self._win = window

    # ---- construction ---------------------------------------------------------
    @classmethod
    def from_host(cls, array, label: str = "", device="cuda",
                  device_buffer: torch.Tensor | None = None) -> "DualView":
        """Adopt host data; the device mirror starts stale (runtime_header.py:119-131).
        ``device_buffer`` adopts an existing device tensor as the mirror (the
        unmanaged-View case)."""
        host = _pinned_like(array)
        if device_buffer is not None:
            if tuple(device_buffer.shape) != tuple(host.shape) or device_buffer.dtype != host.dtype:
                raise ValueError("device_buffer must match the host array's shape and dtype")
            dev = device_buffer
        else:
            dev = torch.empty(host.shape, dtype=host.dtype, device=device)
        rec = _Record(host, dev, label)
        rec.modified_host = True
        return cls(rec)

    @classmethod
    def allocate(cls, shape, dtype, label: str = "", device="cuda") -> "DualView":
        """Both sides allocated, both clean (runtime_header.py:102-117)."""
        host = _pinned_like(torch.zeros(shape, dtype=dtype))
        dev = torch.zeros(shape, dtype=dtype, device=device)
        return cls(_Record(host, dev, label))

    # ---- views ----------------------------------------------------------------
    def host_view(self) -> torch.Tensor:
        self._rec.host_quiescent()
        return self._rec.host if self._win is None else self._rec.host[self._win]

    def device_view(self) -> torch.Tensor:
        return self._rec.device if self._win is None else self._rec.device[self._win]

    def subview(self, *ranges: tuple[int, int]) -> "DualView":
        """Unit-stride window (offset, length) per dim; aliases storage and flags."""
        win = tuple(slice(o, o + n) for o, n in ranges)
        if self._win is not None:
            win = tuple(slice(p.start + w.start, p.start + w.stop) for p, w in zip(self._win, win))
        return DualView(self._rec, win)

    @property
    def shape(self):
        return tuple(self.host_view().shape)

    @property
    def nbytes(self) -> int:
        h = self._rec.host
        return h.numel() * h.element_size()

    def extent(self, r: int) -> int:
        return self.host_view().shape[r]

    def host_modified(self) -> bool:
        return self._rec.modified_host

    def device_modified(self) -> bool:
        return self._rec.modified_device

    # ---- coherence (runtime_header.py:145-178) -----------------------------
    def modify_host(self) -> None:
        self._rec.host_quiescent()
        self._rec.modified_host = True

    def modify_device(self) -> None:
        self._rec.modified_device = True

    def sync_device(self, stream=None) -> None:
        rec = self._rec
        if rec.modified_host:
            with torch.cuda.stream(stream) if stream is not None else _null():
                rec.device.copy_(rec.host, non_blocking=True)
                # the copy stays asynchronous for the device; host-side writers
                # wait on this event (host_view / modify_host)
                rec.h2d_done = torch.cuda.Event()
                rec.h2d_done.record(stream or torch.cuda.current_stream())
            rec.modified_host = False
            _STATS.h2d_count += 1
            _STATS.h2d_bytes += self.nbytes

    def sync_host(self, stream=None) -> None:
        rec = self._rec
        if rec.modified_device:
            with torch.cuda.stream(stream) if stream is not None else _null():
                rec.host.copy_(rec.device, non_blocking=True)
                (stream or torch.cuda.current_stream()).synchronize()
            rec.modified_device = False
            _STATS.d2h_count += 1
            _STATS.d2h_bytes += self.nbytes

    def numpy(self) -> np.ndarray:
        """Host read of the current value (syncs the host side first)."""
        self.sync_host()
        return self.host_view().numpy()


class _null:
    def __enter__(self):
        return None

    def __exit__(self, *a):
        return False
