"""Tensor-level entry points: PyTorch CUDA tensors in, C ABI calls out.

PyTorch is plumbing here (device memory, streams); every operation is one or
more of our sm_100a kernels launched through include/lapis_b200.h on the
tensor's current CUDA stream.  Tensors are passed zero-copy (data_ptr) the way
the reference passes unmanaged Kokkos Views; they must be CUDA, row-major
contiguous (LayoutRight, runtime_header.py:39-41) and of a supported dtype.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _capi
from ._capi import BackendError, check

_DTYPES = {torch.float32: _capi.F32, torch.float64: _capi.F64,
           torch.int32: _capi.I32, torch.int64: _capi.I64}
_COMBINERS = {"add": _capi.ADD, "mul": _capi.MUL, "min": _capi.MIN, "max": _capi.MAX}
_MODES = {"auto": _capi.GEMM_AUTO, "tf32x3": _capi.GEMM_TF32X3, "dmma": _capi.GEMM_DMMA,
          "exact": _capi.GEMM_EXACT, "ozaki": _capi.GEMM_OZAKI}
_initialised: set[int] = set()


def _device_init(t: torch.Tensor) -> None:
    idx = t.device.index if t.device.index is not None else torch.cuda.current_device()
    if idx not in _initialised:
        check(_capi.lib().lapis_b200_init(idx), "lapis_b200_init")
        _initialised.add(idx)


def _from_dlpack(t):
    """A DLPack producer (CuPy, JAX, numba, ... anything with __dlpack__) as a
    zero-copy torch view of the same device memory (tensors via
    DLPack stand in for unmanaged Kokkos Views)."""
    if isinstance(t, torch.Tensor) or not hasattr(t, "__dlpack__"):
        return t
    return torch.from_dlpack(t)


def _dev(t: torch.Tensor, name: str) -> torch.Tensor:
    t = _from_dlpack(t)
    if not isinstance(t, torch.Tensor) or t.device.type != "cuda":
        raise BackendError(f"{name} must be a CUDA tensor (no CPU fallback)", _capi.ERR_ARG)
    if not t.is_contiguous():
        raise BackendError(f"{name} must be row-major contiguous", _capi.ERR_ARG)
    _device_init(t)
    return t


def _dtype(t: torch.Tensor, name: str) -> int:
    if t.dtype not in _DTYPES:
        raise BackendError(f"{name}: unsupported dtype {t.dtype}", _capi.ERR_ARG)
    return _DTYPES[t.dtype]


def _idx_bytes(t: torch.Tensor, name: str) -> int:
    if t.dtype not in (torch.int32, torch.int64):
        raise BackendError(f"{name} must hold int32 or int64 indices", _capi.ERR_ARG)
    return t.element_size()


def _stream(stream) -> C.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t: torch.Tensor | None) -> C.c_void_p:
    return C.c_void_p(t.data_ptr() if t is not None and t.numel() > 0 else None)


def csr_vector_length(nrows: int, nnz: int, max_vector_length: int = 32) -> int:
    """The reference's CSR vector-length hint (loop_mapping.py:224-246)."""
    return int(_capi.lib().lapis_b200_csr_vector_length(nrows, nnz, max_vector_length))


def _check_values(values, x, y):
    if not (values.dtype == x.dtype == y.dtype):
        raise BackendError("values/x/y element types must match (dialect.py:811)", _capi.ERR_ARG)


def _csr_parts(A):
    """(rowptr, colind, values) of a torch.sparse_csr_tensor, zero-copy."""
    if not (isinstance(A, torch.Tensor) and A.layout == torch.sparse_csr):
        raise BackendError("expected a torch.sparse_csr_tensor", _capi.ERR_ARG)
    return A.crow_indices(), A.col_indices(), A.values()


def _is_csr(A) -> bool:
    return isinstance(A, torch.Tensor) and A.layout == torch.sparse_csr


def spmv_csr(rowptr, colind=None, values=None, x=None, y=None, *, vector_length: int = 0,
             nnz: int | None = None, stream=None) -> torch.Tensor:
    """y = A x for CSR A (sparse.spmv_csr, interp.py:798-812).  y is overwritten
    and returned (allocated when None).  ``nnz`` may be passed to avoid reading
    rowptr[N] back from the device.

    Also ``spmv_csr(A, x[, y])`` with A a CUDA ``torch.sparse_csr_tensor``
    (crow / col / values used in place, the ``torch.mv(A_csr, x)`` of
    PAPER.md:298-313).  Any argument may be a DLPack producer."""
    if _is_csr(rowptr):
        A, x, y = rowptr, colind, values
        rowptr, colind, values = _csr_parts(A)
        if nnz is None:
            nnz = A.values().numel()
    rowptr, colind, values, x, y = (_from_dlpack(t) for t in (rowptr, colind, values, x, y))
    for t, n in ((rowptr, "rowptr"), (colind, "colind"), (values, "values"), (x, "x")):
        _dev(t, n)
    nrows = rowptr.numel() - 1
    if y is None:
        y = torch.empty(max(nrows, 0), dtype=values.dtype, device=values.device)
    y = _dev(y, "y")
    _check_values(values, x, y)
    if nrows < 0:
        raise BackendError("rowptr must have at least one entry", _capi.ERR_ARG)
    if y.numel() != nrows:
        raise BackendError(f"y has extent {y.numel()}, rowptr implies {nrows} rows", _capi.ERR_ARG)
    if nnz is None:
        nnz = int(rowptr[-1].item() - rowptr[0].item()) if nrows >= 0 else 0
    check(_capi.lib().lapis_b200_spmv_csr(
        nrows, x.numel(), nnz, _ptr(rowptr), _idx_bytes(rowptr, "rowptr"), _ptr(colind),
        _idx_bytes(colind, "colind"), _ptr(values), _ptr(x), _ptr(y), _dtype(values, "values"),
        vector_length, _stream(stream)), "spmv_csr")
    return y


class CsrPlan:
    """Structure-only analysis of one rowptr (tile -> first-row table), reused
    by every SpMV on that structure.  Holds a device allocation."""

    def __init__(self, rowptr: torch.Tensor, nnz: int | None = None, stream=None,
                 exact: bool | None = None):
        if _is_csr(rowptr):
            rowptr = rowptr.crow_indices()
        rowptr = _dev(rowptr, "rowptr")
        self.nrows = rowptr.numel() - 1
        self.nnz = int(rowptr[-1].item() - rowptr[0].item()) if nnz is None else int(nnz)
        self.rowptr = rowptr
        handle = C.c_void_p()
        check(_capi.lib().lapis_b200_csr_plan_create(
            self.nrows, self.nnz, _ptr(rowptr), _idx_bytes(rowptr, "rowptr"), _stream(stream),
            C.byref(handle)), "csr_plan_create")
        self._handle = handle
        if exact is not None:
            check(_capi.lib().lapis_b200_csr_plan_set_exact(handle, int(bool(exact))),
                  "csr_plan_set_exact")

    def info(self) -> dict:
        """The analysis result: longest row and the kernel the plan dispatches to."""
        out = (C.c_int64 * 4)()
        check(_capi.lib().lapis_b200_csr_plan_info(self._handle, out), "csr_plan_info")
        vl, exact, wb, rs = int(out[1]), bool(out[3] & 1), bool(out[3] & 2), bool(out[3] & 4)
        rs_all = bool(out[3] & 8)
        kind = "exact" if (exact or vl == 1) else "tree (exact for f32)"
        kernel = (f"spmv_vector_kernel<VL={vl}, {kind}>" if vl else "spmv_tile_kernel")
        if rs and (exact or vl == 1):
            kernel = "spmv_rowstream_kernel (exact)"
        elif rs and rs_all:
            kernel = "spmv_rowstream_kernel (reference order, every mode)"
        elif rs:
            kernel = f"spmv_vector_kernel<VL={vl}, tree>; exact / f32: spmv_rowstream_kernel"
        if wb:
            kernel = ("spmv_warpblock_kernel (exact)" if exact else
                      "spmv_warpblock_kernel (rows <= 512 in order, longer: warp tree; f32 exact)")
        return {"max_row_len": int(out[0]), "vector_length": vl, "exact": exact,
                "warpblock": wb, "rowstream": rs, "rowstream_all": rs_all, "ntiles": int(out[2]), "kernel": kernel}

    def spmv(self, colind, values, x, y=None, *, stream=None) -> torch.Tensor:
        colind, values, x, y = (_from_dlpack(t) for t in (colind, values, x, y))
        for t, n in ((colind, "colind"), (values, "values"), (x, "x")):
            _dev(t, n)
        if y is None:
            y = torch.empty(self.nrows, dtype=values.dtype, device=values.device)
        y = _dev(y, "y")
        _check_values(values, x, y)
        check(_capi.lib().lapis_b200_spmv_csr_plan(
            self._handle, _ptr(self.rowptr), _idx_bytes(self.rowptr, "rowptr"), _ptr(colind),
            _idx_bytes(colind, "colind"), _ptr(values), _ptr(x), _ptr(y),
            _dtype(values, "values"), _stream(stream)), "spmv_csr_plan")
        return y

    def close(self) -> None:
        if getattr(self, "_handle", None) is not None and self._handle.value:
            check(_capi.lib().lapis_b200_csr_plan_destroy(self._handle), "csr_plan_destroy")
            self._handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def spmm_csr(rowptr, colind=None, values=None, X=None, Y=None, *, nnz: int | None = None,
             stream=None):
    """Y = A X for CSR A and row-major dense X [ncols, k] (oracle/ir/spmm.mlir).
    Also ``spmm_csr(A, X[, Y])`` with A a CUDA ``torch.sparse_csr_tensor``
    (``torch.sparse.mm(A, X)``); any argument may be a DLPack producer."""
    if _is_csr(rowptr):
        A, X, Y = rowptr, colind, values
        rowptr, colind, values = _csr_parts(A)
        if nnz is None:
            nnz = A.values().numel()
    rowptr, colind, values, X, Y = (_from_dlpack(t) for t in (rowptr, colind, values, X, Y))
    for t, n in ((rowptr, "rowptr"), (colind, "colind"), (values, "values"), (X, "X")):
        _dev(t, n)
    if X.dim() != 2:
        raise BackendError("X must be rank 2", _capi.ERR_ARG)
    nrows = rowptr.numel() - 1
    k = X.shape[1]
    if Y is None:
        Y = torch.empty((nrows, k), dtype=values.dtype, device=values.device)
    Y = _dev(Y, "Y")
    _check_values(values, X, Y)
    if tuple(Y.shape) != (nrows, k):
        raise BackendError(f"Y has shape {tuple(Y.shape)}, expected {(nrows, k)}", _capi.ERR_ARG)
    if nnz is None:
        nnz = int(rowptr[-1].item() - rowptr[0].item())
    check(_capi.lib().lapis_b200_spmm_csr(
        nrows, X.shape[0], nnz, k, _ptr(rowptr), _idx_bytes(rowptr, "rowptr"), _ptr(colind),
        _idx_bytes(colind, "colind"), _ptr(values), _ptr(X), k, _ptr(Y), k,
        _dtype(values, "values"), _stream(stream)), "spmm_csr")
    return Y


class SpmmPlan:
    """Structure-only analysis for repeated Y = A X on one CSR structure
    (lapis_b200_spmm_plan_*): the most referenced rows of X are copied every
    multiply into a compact buffer pinned in L2 (persisting access-policy
    window) and read there through a remapped private colind.  Same results
    as spmm_csr.  ``hot_bytes`` 0 = 16 MB (capped by the device's persisting
    L2 limit)."""

    def __init__(self, rowptr, colind, ncols: int, k: int, dtype=torch.float64, *,
                 nnz: int | None = None, hot_bytes: int = 0, stream=None):
        rowptr, colind = _dev(_from_dlpack(rowptr), "rowptr"), _dev(_from_dlpack(colind), "colind")
        self.nrows = rowptr.numel() - 1
        self.nnz = int(rowptr[-1].item() - rowptr[0].item()) if nnz is None else int(nnz)
        self.k, self.dtype = int(k), dtype
        self.rowptr, self.colind = rowptr, colind
        handle = C.c_void_p()
        check(_capi.lib().lapis_b200_spmm_plan_create(
            self.nrows, int(ncols), self.nnz, self.k, _ptr(rowptr), _idx_bytes(rowptr, "rowptr"),
            _ptr(colind), _idx_bytes(colind, "colind"), _DTYPES[dtype], int(hot_bytes),
            _stream(stream), C.byref(handle)), "spmm_plan_create")
        self._handle = handle

    def info(self) -> dict:
        out = (C.c_int64 * 4)()
        check(_capi.lib().lapis_b200_spmm_plan_info(self._handle, out), "spmm_plan_info")
        far = C.c_int64(0)
        check(_capi.lib().lapis_b200_spmm_plan_hints(self._handle, C.byref(far)), "spmm_plan_hints")
        return {"hot_rows": int(out[0]), "hot_entries": int(out[1]),
                "persisting_bytes": int(out[2]), "nnz": int(out[3]),
                "far_reuse_entries": int(far.value)}

    def spmm(self, values, X, Y=None, *, stream=None) -> torch.Tensor:
        values, X, Y = (_from_dlpack(t) for t in (values, X, Y))
        values, X = _dev(values, "values"), _dev(X, "X")
        if X.dim() != 2 or X.shape[1] != self.k:
            raise BackendError(f"X must be [ncols, {self.k}]", _capi.ERR_ARG)
        if Y is None:
            Y = torch.empty((self.nrows, self.k), dtype=values.dtype, device=values.device)
        Y = _dev(Y, "Y")
        _check_values(values, X, Y)
        check(_capi.lib().lapis_b200_spmm_csr_plan(
            self._handle, _ptr(self.rowptr), _idx_bytes(self.rowptr, "rowptr"), _ptr(self.colind),
            _idx_bytes(self.colind, "colind"), _ptr(values), _ptr(X), X.shape[1], _ptr(Y),
            Y.shape[1], _dtype(values, "values"), _stream(stream)), "spmm_csr_plan")
        return Y

    def close(self) -> None:
        if getattr(self, "_handle", None) is not None and self._handle.value:
            _capi.lib().lapis_b200_spmm_plan_destroy(self._handle)
            self._handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def gemm(A, B, C_out=None, *, mode: str = "auto", stream=None):
    """C = A B (LAPIS::gemm, runtime_header.py:249-266; linalg.matmul)."""
    A = _dev(A, "A"); B = _dev(B, "B")
    if A.dim() != 2 or B.dim() != 2 or A.shape[1] != B.shape[0]:
        raise BackendError(f"matmul shape mismatch {tuple(A.shape)} x {tuple(B.shape)}",
                           _capi.ERR_ARG)
    if A.dtype != B.dtype:
        raise BackendError("element types must match", _capi.ERR_ARG)
    m, k = A.shape
    n = B.shape[1]
    if C_out is None:
        C_out = torch.empty((m, n), dtype=A.dtype, device=A.device)
    C_out = _dev(C_out, "C")
    if tuple(C_out.shape) != (m, n) or C_out.dtype != A.dtype:
        raise BackendError("C has the wrong shape or dtype", _capi.ERR_ARG)
    check(_capi.lib().lapis_b200_gemm(m, n, k, _ptr(A), k, _ptr(B), n, _ptr(C_out), n,
                                      _dtype(A, "A"), _MODES[mode], _stream(stream)), "gemm")
    return C_out


def batch_gemm(A, B, C_out=None, *, mode: str = "auto", stream=None):
    """C[b] = A[b] B[b] (linalg.batch_matmul, interp.py:746-763)."""
    A = _dev(A, "A"); B = _dev(B, "B")
    if A.dim() != 3 or B.dim() != 3 or A.shape[0] != B.shape[0] or A.shape[2] != B.shape[1]:
        raise BackendError("batch_matmul shape mismatch", _capi.ERR_ARG)
    nb, m, k = A.shape
    n = B.shape[2]
    if C_out is None:
        C_out = torch.empty((nb, m, n), dtype=A.dtype, device=A.device)
    C_out = _dev(C_out, "C")
    check(_capi.lib().lapis_b200_batch_gemm(nb, m, n, k, _ptr(A), _ptr(B), _ptr(C_out),
                                            _dtype(A, "A"), _MODES[mode], _stream(stream)),
          "batch_gemm")
    return C_out


def gemv(A, x, y=None, *, stream=None):
    """y = A x (LAPIS::gemv, runtime_header.py:268-282; linalg.matvec)."""
    A = _dev(A, "A"); x = _dev(x, "x")
    if A.dim() != 2 or x.dim() != 1 or A.shape[1] != x.shape[0]:
        raise BackendError("matvec shape mismatch", _capi.ERR_ARG)
    m, n = A.shape
    if y is None:
        y = torch.empty(m, dtype=A.dtype, device=A.device)
    y = _dev(y, "y")
    check(_capi.lib().lapis_b200_gemv(m, n, _ptr(A), n, _ptr(x), _ptr(y), _dtype(A, "A"),
                                      _stream(stream)), "gemv")
    return y


def reduce2d(src, axis: int, combiner: str = "add", out=None, *, stream=None):
    """linalg.reduce over one axis of a rank-2 array (interp.py:779-795)."""
    src = _dev(src, "src")
    if src.dim() != 2:
        raise BackendError("reduce2d expects a rank-2 source", _capi.ERR_ARG)
    rows, cols = src.shape
    if out is None:
        out = torch.empty(rows if axis == 1 else cols, dtype=src.dtype, device=src.device)
    out = _dev(out, "out")
    check(_capi.lib().lapis_b200_reduce_2d(rows, cols, _ptr(src), _ptr(out), axis,
                                           _COMBINERS[combiner], _dtype(src, "src"),
                                           _stream(stream)), "reduce_2d")
    return out


def relu(x, y=None, *, stream=None):
    """y = (x > 0) ? x : 0 (linalg.elementwise cmpf ogt + select)."""
    x = _dev(x, "x")
    if y is None:
        y = torch.empty_like(x)
    y = _dev(y, "y")
    check(_capi.lib().lapis_b200_relu(x.numel(), _ptr(x), _ptr(y), _dtype(x, "x"),
                                      _stream(stream)), "relu")
    return y


def gcn_layer(rowptr, colind, values, X, W, H=None, *, nnz: int | None = None, stream=None,
              exact: bool = False):
    """H = relu((A_hat X) W) — config 4 (oracle/ir/gcn_f32.mlir).  The SpMM stage
    sums in the reference order; the dense stage runs on the tensor cores
    (3xTF32, within 1e-5) unless ``exact`` (reference order: bit-identical).
    A torch.sparse_csr_tensor may be passed for rowptr with colind = values =
    None; any argument may be a DLPack producer."""
    if _is_csr(rowptr):
        rowptr, colind, values = _csr_parts(rowptr)
        if nnz is None:
            nnz = values.numel()
    rowptr, colind, values, X, W, H = (_from_dlpack(t) for t in (rowptr, colind, values, X, W, H))
    for t, nm in ((rowptr, "rowptr"), (colind, "colind"), (values, "values"), (X, "X"), (W, "W")):
        _dev(t, nm)
    if X.dim() != 2 or W.dim() != 2 or X.shape[1] != W.shape[0]:
        raise BackendError("gcn: X [ncols, fin] and W [fin, fout] expected", _capi.ERR_ARG)
    nrows = rowptr.numel() - 1
    if H is None:
        H = torch.empty((nrows, W.shape[1]), dtype=values.dtype, device=values.device)
    H = _dev(H, "H")
    if not (values.dtype == X.dtype == W.dtype == H.dtype):
        raise BackendError("gcn: element types must match", _capi.ERR_ARG)
    if nnz is None:
        nnz = int(rowptr[-1].item() - rowptr[0].item())
    check(_capi.lib().lapis_b200_gcn_layer_mode(
        nrows, X.shape[0], nnz, _ptr(rowptr), _idx_bytes(rowptr, "rowptr"), _ptr(colind),
        _idx_bytes(colind, "colind"), _ptr(values), _ptr(X), X.shape[1], _ptr(W), W.shape[1],
        _ptr(H), _MODES["exact" if exact else "auto"], _dtype(values, "values"), _stream(stream)),
        "gcn_layer")
    return H


def synth_stencil(points: int, n: int, row_begin: int = 0, row_end: int | None = None,
                  device="cuda", stream=None):
    """Generate rows [row_begin, row_end) of the 5-point (2-D) or 27-point (3-D)
    stencil matrix on the device: (rowptr int64 rebased, colind int32, values f64)."""
    N = n * n if points == 5 else n ** 3
    row_end = N if row_end is None else row_end
    rows = row_end - row_begin
    rowptr = torch.empty(rows + 1, dtype=torch.int64, device=device)
    rowptr = _dev(rowptr, "rowptr")
    check(_capi.lib().lapis_b200_synth_stencil(points, n, row_begin, row_end, _ptr(rowptr), None,
                                               None, _stream(stream)), "synth_stencil(rowptr)")
    nnz = int(rowptr[-1].item())
    colind = torch.empty(nnz, dtype=torch.int32, device=device)
    values = torch.empty(nnz, dtype=torch.float64, device=device)
    check(_capi.lib().lapis_b200_synth_stencil(points, n, row_begin, row_end, _ptr(rowptr),
                                               _ptr(colind), _ptr(values), _stream(stream)),
          "synth_stencil")
    return rowptr, colind, values
