"""ctypes front of oracle/lapis_oracle.c — the CPU restatement of the reference
semantics.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Every function mirrors a reference handler (file:line cited in the C source)
and returns numpy arrays; row loops run on OpenMP threads without changing any
per-row summation order.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from . import build as _build

F32, F64, I32, I64 = 0, 1, 2, 3
_DT = {np.dtype(np.float32): F32, np.dtype(np.float64): F64,
       np.dtype(np.int32): I32, np.dtype(np.int64): I64}
COMBINERS = {"add": 0, "mul": 1, "min": 2, "max": 3}

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        so = _build.ORACLE_SO
        if not so.exists():
            _build.build_oracle()
        _lib = C.CDLL(str(so))
        i64, vp, ci = C.c_int64, C.c_void_p, C.c_int
        _lib.oracle_csr_vector_length.restype = i64
        _lib.oracle_csr_vector_length.argtypes = [i64, i64, i64]
        _lib.oracle_max_threads.restype = ci
        _lib.oracle_spmv_csr.argtypes = [i64, i64, vp, ci, vp, ci, vp, vp, vp, ci, ci]
        _lib.oracle_spmm_csr.argtypes = [i64, i64, i64, vp, ci, vp, ci, vp, vp, i64, vp, i64, ci, ci]
        _lib.oracle_matmul.argtypes = [i64, i64, i64, vp, i64, vp, i64, vp, i64, ci, ci]
        _lib.oracle_matmul_entries.argtypes = [i64, vp, i64, vp, i64, i64, vp, vp, vp, ci, ci]
        _lib.oracle_matvec.argtypes = [i64, i64, vp, i64, vp, vp, ci, ci]
        _lib.oracle_batch_matmul.argtypes = [i64, i64, i64, i64, vp, vp, vp, ci, ci]
        _lib.oracle_reduce2d.argtypes = [i64, i64, vp, vp, ci, ci, ci, ci]
        _lib.oracle_relu.argtypes = [i64, vp, vp, ci]
    return _lib


def _p(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


def _c(a, dtype=None):
    return np.ascontiguousarray(a if dtype is None else np.asarray(a, dtype=dtype))


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def csr_vector_length(nrows: int, nnz: int, cap: int = 32) -> int:
    """loop_mapping.py:224-246 — the CSR vector-length hint."""
    return int(lib().oracle_csr_vector_length(nrows, nnz, cap))


def spmv_csr(rowptr, colind, values, x, rows=None, threads=0) -> np.ndarray:
    """interp.py:798-812; rows=(r0, r1) restricts to a row range (y has r1-r0 entries
    filled at their global positions in a length-nrows array)."""
    rowptr, colind, values, x = _c(rowptr), _c(colind), _c(values), _c(x)
    n = rowptr.shape[0] - 1
    r0, r1 = rows if rows is not None else (0, n)
    y = np.zeros(n, dtype=values.dtype)
    lib().oracle_spmv_csr(r0, r1, _p(rowptr), rowptr.itemsize, _p(colind), colind.itemsize,
                          _p(values), _p(x), _p(y), _DT[values.dtype], threads)
    return y


def spmm_csr(rowptr, colind, values, X, rows=None, threads=0) -> np.ndarray:
    rowptr, colind, values, X = _c(rowptr), _c(colind), _c(values), _c(X)
    n = rowptr.shape[0] - 1
    k = X.shape[1]
    r0, r1 = rows if rows is not None else (0, n)
    Y = np.zeros((n, k), dtype=values.dtype)
    lib().oracle_spmm_csr(r0, r1, k, _p(rowptr), rowptr.itemsize, _p(colind), colind.itemsize,
                          _p(values), _p(X), k, _p(Y), k, _DT[values.dtype], threads)
    return Y


def matmul(A, B, threads=0) -> np.ndarray:
    """interp.py:711-722."""
    A, B = _c(A), _c(B)
    m, k = A.shape
    n = B.shape[1]
    Cm = np.zeros((m, n), dtype=A.dtype)
    lib().oracle_matmul(m, n, k, _p(A), k, _p(B), n, _p(Cm), n, _DT[A.dtype], threads)
    return Cm


def matmul_entries(A, B, ii, jj, threads=0) -> np.ndarray:
    A, B = _c(A), _c(B)
    ii, jj = _c(ii, np.int64), _c(jj, np.int64)
    out = np.zeros(ii.shape[0], dtype=A.dtype)
    lib().oracle_matmul_entries(A.shape[1], _p(A), A.shape[1], _p(B), B.shape[1], ii.shape[0],
                                _p(ii), _p(jj), _p(out), _DT[A.dtype], threads)
    return out


def matvec(A, x, threads=0) -> np.ndarray:
    """interp.py:729-739."""
    A, x = _c(A), _c(x)
    m, n = A.shape
    y = np.zeros(m, dtype=A.dtype)
    lib().oracle_matvec(m, n, _p(A), n, _p(x), _p(y), _DT[A.dtype], threads)
    return y


def batch_matmul(A, B, threads=0) -> np.ndarray:
    """interp.py:746-763."""
    A, B = _c(A), _c(B)
    nb, m, k = A.shape
    n = B.shape[2]
    Cm = np.zeros((nb, m, n), dtype=A.dtype)
    lib().oracle_batch_matmul(nb, m, n, k, _p(A), _p(B), _p(Cm), _DT[A.dtype], threads)
    return Cm


def reduce2d(src, axis: int, combiner: str, threads=0) -> np.ndarray:
    """interp.py:779-795 for a rank-2 source and one reduced axis."""
    src = _c(src)
    rows, cols = src.shape
    out = np.zeros(rows if axis == 1 else cols, dtype=src.dtype)
    lib().oracle_reduce2d(rows, cols, _p(src), _p(out), axis, COMBINERS[combiner],
                          _DT[src.dtype], threads)
    return out


def relu(x) -> np.ndarray:
    x = _c(x)
    y = np.empty_like(x)
    lib().oracle_relu(x.size, _p(x), _p(y), _DT[x.dtype])
    return y


def gcn(rowptr, colind, values, X, W, threads=0) -> np.ndarray:
    """relu((A_hat X) W) in the reference order: SpMM, matmul, elementwise select."""
    return relu(matmul(spmm_csr(rowptr, colind, values, X, threads=threads), W, threads=threads))


def diff_outputs(a: list, b: list, rel_tol: float = 1e-12):
    """interp.py:1050-1071: ints exact; floats |x-y| <= rel_tol*max(|x|,|y|,1).
    Returns (match, message)."""
    if len(a) != len(b):
        return False, f"output arity {len(a)} vs {len(b)}"
    for i, (x, y) in enumerate(zip(a, b)):
        xa, ya = np.asarray(x), np.asarray(y)
        if xa.shape != ya.shape:
            return False, f"output {i}: shape {xa.shape} vs {ya.shape}"
        if xa.dtype.kind in "iub" and ya.dtype.kind in "iub":
            if not np.array_equal(xa, ya):
                bad = np.argwhere(xa != ya)[0]
                return False, f"output {i} at {tuple(int(v) for v in bad)}: {xa[tuple(bad)]} vs {ya[tuple(bad)]}"
        else:
            xf, yf = xa.astype(np.float64), ya.astype(np.float64)
            tol = rel_tol * np.maximum(np.maximum(np.abs(xf), np.abs(yf)), 1.0)
            ok = np.abs(xf - yf) <= tol
            if not np.all(ok):
                bad = np.argwhere(~ok)[0]
                return False, f"output {i} at {tuple(int(v) for v in bad)}: {xf[tuple(bad)]} vs {yf[tuple(bad)]}"
    return True, "match"
