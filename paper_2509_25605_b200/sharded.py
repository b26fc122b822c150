"""Row-block-sharded CSR SpMV across GPUs.

One process per GPU (torch.distributed, NCCL).  Rank r owns the contiguous
rows [row_begin, row_end) — rowptr rebased to 0, colind kept GLOBAL — and the
matching slice of x and y.  The only exchange step of the path is x: each rank
needs the x entries of the columns its rows reference.  Instead of gathering
all of x, the plan records, per peer, the contiguous column interval this rank
reads from that peer's rows (for a stencil the two halo slabs of
n^2 + n + 1 rows) and every step moves exactly those slabs with NCCL P2P
(batch_isend_irecv) on a communication stream — an allgather restricted to the
needed span.

Overlap: local rows are split into an interior run (every column owned
locally, computed while the exchange is in flight) and the boundary rows
before / after it (computed once the slabs have landed).  Rows are never
split, so each y entry is still the reference's ascending sequential sum —
the sharded result is bit-identical to the single-GPU one.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


def balanced_row_ranges(nrows: int, world: int) -> list[tuple[int, int]]:
    """Contiguous row blocks of (near) equal row count."""
    return [(nrows * r // world, nrows * (r + 1) // world) for r in range(world)]


def balanced_nnz_ranges(rowptr_global_ends, nrows: int, world: int) -> list[tuple[int, int]]:
    """Contiguous row blocks balanced by nonzeros, from a host int64 rowptr."""
    import numpy as np
    rp = np.asarray(rowptr_global_ends)
    total = int(rp[-1] - rp[0])
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(rp, rp[0] + total * r // world, side="left")))
    cuts.append(nrows)
    return [(cuts[i], cuts[i + 1]) for i in range(world)]


@dataclass
class ExchangePlan:
    """needs[p] = (lo, hi): global x columns this rank reads from peer p
    (empty when lo >= hi); sends[p] = (lo, hi): columns of this rank's rows
    that peer p reads."""
    rank: int
    world: int
    ranges: list[tuple[int, int]]
    needs: list[tuple[int, int]]
    sends: list[tuple[int, int]]

    @property
    def recv_elems(self) -> int:
        return sum(max(0, hi - lo) for p, (lo, hi) in enumerate(self.needs) if p != self.rank)

    @property
    def send_elems(self) -> int:
        return sum(max(0, hi - lo) for p, (lo, hi) in enumerate(self.sends) if p != self.rank)


def column_needs(colind: torch.Tensor, ranges: list[tuple[int, int]]) -> list[tuple[int, int]]:
    """Per owner p, the [min, max+1) interval of referenced columns inside p's rows."""
    out = []
    for lo, hi in ranges:
        m = (colind >= lo) & (colind < hi)
        if bool(m.any()):
            sel = colind[m]
            out.append((int(sel.min()), int(sel.max()) + 1))
        else:
            out.append((0, 0))
    return out


def build_exchange_plan(colind: torch.Tensor, ranges, rank: int, world: int,
                        group=None) -> ExchangePlan:
    needs = column_needs(colind, ranges)
    if world == 1:
        return ExchangePlan(rank, world, list(ranges), needs, [(0, 0)])
    dev = colind.device if dist.get_backend(group) == "nccl" else torch.device("cpu")
    mine = torch.tensor([v for lo_hi in needs for v in lo_hi], dtype=torch.int64, device=dev)
    allv = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(allv, mine, group=group)
    sends = []
    for p in range(world):
        v = allv[p].cpu().tolist()
        sends.append((v[2 * rank], v[2 * rank + 1]))
    return ExchangePlan(rank, world, list(ranges), needs, sends)


def exchange(plan: ExchangePlan, x_full: torch.Tensor, group=None):
    """Post the halo slabs (P2P) — returns the request list; x_full is indexed by
    GLOBAL column and already holds this rank's own slice."""
    if x_full.is_cuda and dist.get_backend(group) == "gloo":
        return _exchange_staged(plan, x_full, group)
    ops = []
    for p in range(plan.world):
        if p == plan.rank:
            continue
        lo, hi = plan.sends[p]
        if hi > lo:
            ops.append(dist.P2POp(dist.isend, x_full[lo:hi], p, group=group))
        lo, hi = plan.needs[p]
        if hi > lo:
            ops.append(dist.P2POp(dist.irecv, x_full[lo:hi], p, group=group))
    return dist.batch_isend_irecv(ops) if ops else []


def _exchange_staged(plan: ExchangePlan, x_full: torch.Tensor, group=None):
    """gloo moves host tensors only: the same slabs through host copies,
    completed before returning (correctness runs of the N > 1 path on one
    GPU; the product path is NCCL)."""
    ops, staged = [], []
    for p in range(plan.world):
        if p == plan.rank:
            continue
        lo, hi = plan.sends[p]
        if hi > lo:
            ops.append(dist.P2POp(dist.isend, x_full[lo:hi].cpu(), p, group=group))
        lo, hi = plan.needs[p]
        if hi > lo:
            buf = torch.empty_like(x_full[lo:hi], device="cpu")
            ops.append(dist.P2POp(dist.irecv, buf, p, group=group))
            staged.append((lo, hi, buf))
    for r in (dist.batch_isend_irecv(ops) if ops else []):
        r.wait()
    for lo, hi, buf in staged:
        x_full[lo:hi].copy_(buf)
    return []


def interior_run(rowptr: torch.Tensor, colind: torch.Tensor, own: tuple[int, int]) -> tuple[int, int]:
    """Longest run [a, b) of local rows whose columns all lie in `own`."""
    nloc = rowptr.numel() - 1
    if nloc == 0:
        return 0, 0
    remote = ((colind < own[0]) | (colind >= own[1])).to(torch.int64)
    # per-row count of remote references via prefix sums over the nnz stream
    csum = torch.zeros(colind.numel() + 1, dtype=torch.int64, device=colind.device)
    csum[1:] = torch.cumsum(remote, 0)
    base = rowptr[0]
    per_row = csum[(rowptr[1:] - base)] - csum[(rowptr[:-1] - base)]
    ones = torch.nonzero(per_row > 0).flatten().cpu()
    pos = torch.cat([torch.tensor([-1]), ones, torch.tensor([nloc])])
    gaps = pos[1:] - pos[:-1] - 1
    i = int(torch.argmax(gaps))
    a = int(pos[i]) + 1
    return a, a + int(gaps[i])


class RowBlockSpmv:
    """y_local = A[row_begin:row_end, :] x with the halo exchange overlapped."""

    def __init__(self, rowptr: torch.Tensor, colind: torch.Tensor, values: torch.Tensor,
                 row_begin: int, row_end: int, nrows_global: int, ranges, rank: int, world: int,
                 group=None, exact: bool | None = None):
        from .kernels import CsrPlan
        self.rowptr, self.colind, self.values = rowptr, colind, values
        self.row_begin, self.row_end = row_begin, row_end
        self.rank, self.world, self.group = rank, world, group
        self.plan = build_exchange_plan(colind, ranges, rank, world, group)
        a, b = interior_run(rowptr, colind, (row_begin, row_end)) if world > 1 else (0, row_end - row_begin)
        self.interior = (a, b)
        nloc = row_end - row_begin
        self.pieces = [(0, a), (a, b), (b, nloc)]
        self.plans = {}
        for lo, hi in self.pieces:
            if hi > lo:
                rp = rowptr[lo:hi + 1]
                self.plans[(lo, hi)] = CsrPlan(rp, exact=exact)
        self.comm_stream = torch.cuda.Stream(device=values.device) if world > 1 else None

    @property
    def launches_per_multiply(self) -> int:
        return len(self.plans)

    def multiply(self, x_full: torch.Tensor, y_local: torch.Tensor, stream=None) -> torch.Tensor:
        stream = stream or torch.cuda.current_stream()
        a, b = self.interior
        reqs = []
        if self.world > 1:
            self.comm_stream.wait_stream(stream)
            with torch.cuda.stream(self.comm_stream):
                reqs = exchange(self.plan, x_full, self.group)
        if b > a:
            self.plans[(a, b)].spmv(self.colind, self.values, x_full, y_local[a:b], stream=stream)
        # r.wait() makes the CURRENT stream wait on the NCCL work, so it runs
        # under the caller's stream: the boundary rows below are ordered after
        # the slabs even when `stream` is not the current stream
        with torch.cuda.stream(stream):
            for r in reqs:
                r.wait()
        if self.world > 1:
            stream.wait_stream(self.comm_stream)
        for lo, hi in ((0, a), (b, y_local.numel())):
            if hi > lo:
                self.plans[(lo, hi)].spmv(self.colind, self.values, x_full, y_local[lo:hi],
                                          stream=stream)
        return y_local


# --------------------------------------------------------------------- SpMM
def equal_row_ranges(nrows: int, world: int) -> list[tuple[int, int]]:
    """Row blocks of exactly ceil(nrows / world) rows (the last one shorter), so
    that every rank's block occupies the same-sized slot of an all-gathered
    buffer and a GLOBAL row index addresses that buffer directly."""
    c = -(-nrows // world) if world > 0 else 0
    return [(min(nrows, r * c), min(nrows, (r + 1) * c)) for r in range(world)]


class RowBlockSpmm:
    """Y_local = A[row_begin:row_end, :] X for a row-sharded dense operand X
    (SURVEY 8(e), config 3 / the GCN features): rank r owns the rows
    [r*c, r*c + c) of A, X and Y (c = ceil(N / world)), colind stays GLOBAL.

    The exchange step is one NCCL all-gather of X into a [world*c, k] buffer
    (in place: this rank's slot is the send buffer), after which the local
    SpMM kernel reads any X row by its global index.  A power-law matrix
    references essentially every column from every shard, so the halo
    exchange of RowBlockSpmv would degenerate into the same all-gather; the
    collective is used directly (NVLS-capable over NVSwitch).  Rows are never
    split, so every Y entry is the reference's ascending sum (bit-identical to
    one GPU)."""

    def __init__(self, rowptr: torch.Tensor, colind: torch.Tensor, values: torch.Tensor,
                 nrows_global: int, k: int, rank: int, world: int, group=None, plan: bool = False,
                 hot_bytes: int = 0):
        self.rowptr, self.colind, self.values = rowptr, colind, values
        self.N, self.k, self.rank, self.world, self.group = nrows_global, k, rank, world, group
        self.ranges = equal_row_ranges(nrows_global, world)
        self.row_begin, self.row_end = self.ranges[rank]
        self.chunk = -(-nrows_global // world)
        self.nnz = int(rowptr[-1].item() - rowptr[0].item())
        self.X_full = torch.zeros((world * self.chunk, k), dtype=values.dtype,
                                  device=values.device)
        self.plan = None
        if plan and values.is_cuda:
            from .kernels import SpmmPlan
            self.plan = SpmmPlan(rowptr, colind, nrows_global, k, values.dtype, nnz=self.nnz,
                                 hot_bytes=hot_bytes)

    @property
    def x_local(self) -> torch.Tensor:
        """This rank's rows of X (write them here before a multiply)."""
        return self.X_full[self.rank * self.chunk:self.rank * self.chunk
                           + (self.row_end - self.row_begin)]

    @property
    def gather_bytes(self) -> int:
        """Bytes this rank receives per all-gather."""
        return (self.world - 1) * self.chunk * self.k * self.X_full.element_size()

    def gather(self) -> None:
        if self.world > 1:
            slot = self.X_full[self.rank * self.chunk:(self.rank + 1) * self.chunk]
            if self.X_full.is_cuda and dist.get_backend(self.group) == "gloo":
                host = self.X_full.cpu()   # correctness runs on one GPU (gloo)
                dist.all_gather_into_tensor(host, slot.cpu(), group=self.group)
                self.X_full.copy_(host)
                return
            dist.all_gather_into_tensor(self.X_full, slot, group=self.group)

    def multiply(self, Y_local: torch.Tensor, stream=None, replicated: bool = False):
        """All-gather X (unless it is already replicated), then the local SpMM."""
        from .kernels import spmm_csr
        if not replicated:
            self.gather()
        if self.plan is not None:
            return self.plan.spmm(self.values, self.X_full[:self.N], Y_local, stream=stream)
        return spmm_csr(self.rowptr, self.colind, self.values, self.X_full[:self.N], Y_local,
                        nnz=self.nnz, stream=stream)


# ------------------------------------------------------------ dense GEMM
class RowBlockGemm:
    """C[r0:r1, :] = A[r0:r1, :] B on rank r: the rows
    of A and C are sharded in equal blocks (equal_row_ranges), B is replicated
    by ONE broadcast from rank 0 when the operator is built — outside any
    steady-state step, and stated as such in the bench line.  The step itself
    has no collective: every C row is computed whole on one GPU, so C is
    bit-identical to the one-GPU product for every mode (the k order of an
    output element does not depend on the row blocking).  ``gather_c`` is the
    optional all-gather of C (not part of the step)."""

    def __init__(self, A_local: torch.Tensor, B: torch.Tensor, m_global: int, rank: int,
                 world: int, group=None, src: int = 0):
        self.A_local, self.B = A_local, B
        self.m, self.rank, self.world, self.group = m_global, rank, world, group
        self.ranges = equal_row_ranges(m_global, world)
        self.row_begin, self.row_end = self.ranges[rank]
        if A_local.shape[0] != self.row_end - self.row_begin:
            raise ValueError("A_local must hold this rank's row block")
        self.broadcast_bytes = B.numel() * B.element_size()
        if world > 1:
            if B.is_cuda and dist.get_backend(group) == "gloo":
                host = B.cpu()
                dist.broadcast(host, src, group=group)
                B.copy_(host)
            else:
                dist.broadcast(B, src, group=group)

    def multiply(self, C_local: torch.Tensor, mode: str = "auto", stream=None) -> torch.Tensor:
        from .kernels import gemm
        return gemm(self.A_local, self.B, C_local, mode=mode, stream=stream)

    def gather_c(self, C_local: torch.Tensor) -> torch.Tensor:
        c = -(-self.m // self.world)
        full = torch.zeros((self.world * c, C_local.shape[1]), dtype=C_local.dtype,
                           device=C_local.device)
        slot = full[self.rank * c:self.rank * c + C_local.shape[0]]
        slot.copy_(C_local)
        if self.world > 1:
            mine = full[self.rank * c:(self.rank + 1) * c]
            if full.is_cuda and dist.get_backend(self.group) == "gloo":
                host = full.cpu()
                dist.all_gather_into_tensor(host, mine.cpu(), group=self.group)
                full.copy_(host)
            else:
                dist.all_gather_into_tensor(full, mine, group=self.group)
        return full[:self.m]


# ------------------------------------------------------------- GCN layer
class RowBlockGcn:
    """H[r0:r1] = relu((A_hat[r0:r1, :] X) W) on rank r:
    A_hat and H in row blocks, X row-sharded like RowBlockSpmm (one NCCL
    all-gather of the features per step, the layer's only exchange), W
    replicated (broadcast once from rank 0 at construction).  Each H row is
    computed whole on one GPU (bit-identical to one GPU)."""

    def __init__(self, rowptr: torch.Tensor, colind: torch.Tensor, values: torch.Tensor,
                 W: torch.Tensor, nrows_global: int, rank: int, world: int, group=None):
        self.spmm = RowBlockSpmm(rowptr, colind, values, nrows_global, W.shape[0], rank, world,
                                 group)
        self.W, self.rank, self.world, self.group = W, rank, world, group
        self.row_begin, self.row_end = self.spmm.row_begin, self.spmm.row_end
        if world > 1:
            if W.is_cuda and dist.get_backend(group) == "gloo":
                host = W.cpu()
                dist.broadcast(host, 0, group=group)
                W.copy_(host)
            else:
                dist.broadcast(W, 0, group=group)

    @property
    def x_local(self) -> torch.Tensor:
        return self.spmm.x_local

    @property
    def gather_bytes(self) -> int:
        return self.spmm.gather_bytes

    def gather(self) -> None:
        self.spmm.gather()

    def multiply(self, H_local: torch.Tensor, stream=None, replicated: bool = False):
        from .kernels import gcn_layer
        if not replicated:
            self.gather()
        sp = self.spmm
        return gcn_layer(sp.rowptr, sp.colind, sp.values, sp.X_full[:sp.N], self.W, H_local,
                         nnz=sp.nnz, stream=stream)


# ------------------------------------------------- native (C-ABI) row blocks
class NcclComm:
    """A communicator of the backend's own (lapis_b200_nccl_comm_init): rank 0
    draws the NCCL unique id, the process group broadcasts its 128 bytes."""

    def __init__(self, rank: int, world: int, group=None):
        import ctypes as C
        from . import _capi
        from ._capi import check
        uid = (C.c_char * 128)()
        if rank == 0:
            check(_capi.lib().lapis_b200_nccl_unique_id(uid), "nccl_unique_id")
        if world > 1:
            t = torch.tensor(list(bytes(uid)), dtype=torch.uint8)
            if dist.get_backend(group) == "nccl":
                t = t.cuda()
            dist.broadcast(t, 0, group=group)
            uid = (C.c_char * 128).from_buffer_copy(bytes(t.cpu().tolist()))
        handle = C.c_void_p()
        check(_capi.lib().lapis_b200_nccl_comm_init(uid, world, rank, C.byref(handle)),
              "nccl_comm_init")
        self.handle, self.rank, self.world = handle, rank, world

    def close(self) -> None:
        from . import _capi
        if getattr(self, "handle", None) is not None and self.handle.value:
            _capi.lib().lapis_b200_nccl_comm_destroy(self.handle)
            self.handle = None


class NativeRowBlockSpmv:
    """RowBlockSpmv through the C ABI (lapis_b200_rowblock_*): the same
    exchange plan, interior/boundary split and overlap, run natively with the
    backend's own NCCL communicator.  rowptr rebased to 0, colind global."""

    def __init__(self, rowptr: torch.Tensor, colind: torch.Tensor, values: torch.Tensor,
                 ranges, rank: int, world: int, comm: NcclComm | None = None,
                 exact: bool = False, stream=None):
        import ctypes as C
        from . import _capi
        from ._capi import check
        from .kernels import _idx_bytes, _ptr, _stream
        self.rowptr, self.colind, self.values = rowptr, colind, values
        self.rank, self.world = rank, world
        begins = (C.c_int64 * (world + 1))(*([lo for lo, _ in ranges] + [ranges[-1][1]]))
        nnz = int(rowptr[-1].item())
        handle = C.c_void_p()
        check(_capi.lib().lapis_b200_rowblock_create(
            comm.handle if comm is not None else None, rank, world, begins, _ptr(rowptr),
            _idx_bytes(rowptr, "rowptr"), _ptr(colind), _idx_bytes(colind, "colind"), nnz,
            int(bool(exact)), _stream(stream), C.byref(handle)), "rowblock_create")
        self._handle = handle

    def info(self) -> dict:
        import ctypes as C
        from . import _capi
        from ._capi import check
        out = (C.c_int64 * (2 + 4 * self.world))()
        check(_capi.lib().lapis_b200_rowblock_info(self._handle, out), "rowblock_info")
        v = list(out)
        return {"interior": (v[0], v[1]),
                "needs": [(v[2 + 4 * p], v[3 + 4 * p]) for p in range(self.world)],
                "sends": [(v[4 + 4 * p], v[5 + 4 * p]) for p in range(self.world)]}

    def multiply(self, x_full: torch.Tensor, y_local: torch.Tensor, stream=None) -> torch.Tensor:
        from . import _capi
        from ._capi import check
        from .kernels import _dtype, _idx_bytes, _ptr, _stream
        check(_capi.lib().lapis_b200_spmv_csr_rowblock(
            self._handle, _ptr(self.rowptr), _idx_bytes(self.rowptr, "rowptr"), _ptr(self.colind),
            _idx_bytes(self.colind, "colind"), _ptr(self.values), _ptr(x_full), _ptr(y_local),
            _dtype(self.values, "values"), _stream(stream)), "spmv_csr_rowblock")
        return y_local

    def close(self) -> None:
        from . import _capi
        if getattr(self, "_handle", None) is not None and self._handle.value:
            _capi.lib().lapis_b200_rowblock_destroy(self._handle)
            self._handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
