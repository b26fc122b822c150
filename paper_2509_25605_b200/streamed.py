"""SpMV on host-resident vectors with the transfers hidden behind the kernels.

The reference's calling convention keeps x and y in DualViews: the emitted
``spmv`` syncs x to the device, runs the kernel and marks y device-modified;
reading y on the host syncs it back (golden cpp/spmv.hpp:34-68,
runtime_header.py:145-178).  Done literally that is H2D(all of x) ->
SpMV -> D2H(all of y), three serialised phases dominated by the host link.

``StreamedSpmv`` keeps those semantics (after ``multiply`` x is synced, y is
synced back to the host; one H2D and one D2H in ``transfer_stats``) but cuts
the work into row chunks balanced by nonzeros:

* the H2D of x runs on its own stream in column order, in pieces ending where
  each row chunk's columns end (a structure-only analysis: the prefix maximum
  of every chunk's largest column), so chunk i starts as soon as the x it
  reads is resident;
* chunk i's SpMV runs on the compute stream (its own CsrPlan), then its slice
  of y goes back on a third stream while chunk i+1 computes.

For banded matrices (the stencils of configs 1 and 5) the host link carries x
in and y out concurrently (full duplex) and the kernels run in the shadow of
the copies; for matrices whose chunks read all of x the copy of x simply
completes before the first chunk.  Results are those of the plan kernels
(bit-identical in exact mode).
"""
from __future__ import annotations

import os

import torch

from . import dualview as _dv
from .dualview import DualView
from .kernels import CsrPlan, _dev


class StreamedSpmv:
    def __init__(self, rowptr: torch.Tensor, colind: torch.Tensor, values: torch.Tensor,
                 ncols: int, chunks: int | None = None, exact: bool | None = None):
        for t, n in ((rowptr, "rowptr"), (colind, "colind"), (values, "values")):
            _dev(t, n)
        self.rowptr, self.colind, self.values = rowptr, colind, values
        self.ncols = int(ncols)
        nrows = rowptr.numel() - 1
        base = int(rowptr[0].item())
        nnz = int(rowptr[-1].item()) - base
        if chunks is None:   # ~256 MB of matrix per chunk, at most 16 chunks
            env = os.environ.get("LAPIS_B200_STREAM_CHUNKS")
            cap = int(env) if env else 16
            chunks = min(cap, max(1, (nnz * (values.element_size() + colind.element_size())) >> 28))
        chunks = max(1, min(chunks, nrows))
        # row boundaries at equal nonzero counts
        targets = torch.tensor([base + (nnz * c) // chunks for c in range(1, chunks)],
                               dtype=rowptr.dtype, device=rowptr.device)
        cuts = torch.searchsorted(rowptr, targets).clamp_(0, nrows).cpu().tolist() if chunks > 1 else []
        bounds = sorted(set([0, *cuts, nrows]))
        self.ranges = [(lo, hi) for lo, hi in zip(bounds[:-1], bounds[1:]) if hi > lo]
        self.plans = [CsrPlan(rowptr[lo:hi + 1], exact=exact) for lo, hi in self.ranges]
        # structure analysis: x prefix each chunk needs (prefix max of its largest column + 1)
        need, hi_so_far = [], 0
        for lo, hi in self.ranges:
            a, b = int(rowptr[lo].item()) - 0, int(rowptr[hi].item())
            cmax = int(colind[a:b].max().item()) + 1 if b > a else 0
            hi_so_far = min(self.ncols, max(hi_so_far, cmax))
            need.append(hi_so_far)
        self.need = need
        dev = values.device
        self.h2d = torch.cuda.Stream(device=dev)
        self.d2h = torch.cuda.Stream(device=dev)

    @property
    def launches_per_multiply(self) -> int:
        return len(self.plans)

    def multiply(self, x: DualView, y: DualView, stream=None) -> None:
        """y = A x; x and y are DualViews (x: ncols, y: nrows).  On return x
        is synced to the device and y's host copy holds the result."""
        compute = stream or torch.cuda.current_stream()
        xh, xd = x.host_view(), x.device_view()
        yh, yd = y.host_view(), y.device_view()
        ready = []
        copy_x = x.host_modified()
        if copy_x:
            self.h2d.wait_stream(compute)     # the previous users of x's device buffer
            done = 0
            with torch.cuda.stream(self.h2d):
                for hi in self.need:
                    if hi > done:
                        xd[done:hi].copy_(xh[done:hi], non_blocking=True)
                        done = hi
                    ev = torch.cuda.Event()
                    ev.record(self.h2d)
                    ready.append(ev)
                if done < self.ncols:          # the rest: the whole buffer is synced
                    xd[done:].copy_(xh[done:], non_blocking=True)
        self.d2h.wait_stream(compute)
        for i, ((lo, hi), plan) in enumerate(zip(self.ranges, self.plans)):
            if copy_x:
                compute.wait_event(ready[i])
            plan.spmv(self.colind, self.values, xd, yd[lo:hi], stream=compute)
            ev = torch.cuda.Event()
            ev.record(compute)
            self.d2h.wait_event(ev)
            with torch.cuda.stream(self.d2h):
                yh[lo:hi].copy_(yd[lo:hi], non_blocking=True)
        if copy_x:
            compute.wait_stream(self.h2d)
            x._rec.modified_host = False
            _dv._STATS.h2d_count += 1
            _dv._STATS.h2d_bytes += x.nbytes
        self.d2h.synchronize()                # y's host copy is what the caller reads next
        if copy_x:
            self.h2d.synchronize()            # x's host side may be rewritten on return
        compute.wait_stream(self.d2h)
        y._rec.modified_device = False
        _dv._STATS.d2h_count += 1
        _dv._STATS.d2h_bytes += y.nbytes
