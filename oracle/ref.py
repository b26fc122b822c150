"""ctypes front of oracle/_ref/liblapis_ref.so — the reference's OWN emitted
Kokkos C++ for the hot kernels, running on the reference's OWN serial Kokkos
stub (built by oracle/build.py).  TEST / BASELINE INFRASTRUCTURE ONLY.

Each call returns (output, seconds) where ``seconds`` is a numpy array with the
wall time of each of `reps` calls of the emitted function, taken after one
warm-up call (the warm-up performs the lazy host->"device" DualView copies, as
in the reference).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import build as _build

_lib = None


def available() -> bool:
    return _build.REF_SO.exists() or _build.REF_SO_NATIVE.exists()


def variant() -> str:
    """Which build runs: the -march=native one when this host's CPU has every
    ISA flag of the build host, else the portable (-O3, baseline x86-64) one."""
    so = _build.REF_SO_NATIVE
    if so.exists() and _build.NATIVE_FLAGS.exists():
        need = set(_build.NATIVE_FLAGS.read_text().split())
        if need and need <= _build.cpu_flags():
            return "native"
    return "portable"


def compile_flags() -> str:
    return ("g++ -O3 -march=native (build host) -ffp-contract=off" if variant() == "native"
            else "g++ -O3 -ffp-contract=off (portable: this CPU lacks an ISA flag of the build host)")


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not available():
            _build.build_reference()
        if not available():
            raise RuntimeError("reference CPU path not built (needs /root/reference once)")
        so = _build.REF_SO_NATIVE if variant() == "native" else _build.REF_SO
        _lib = C.CDLL(str(so))
        i64, vp, ci = C.c_int64, C.c_void_p, C.c_int
        for name in ("ref_spmv_f64_i64", "ref_spmv_f64_i32", "ref_spmm_f64_i32", "ref_gcn_f32_i32"):
            f = getattr(_lib, name)
            f.argtypes = [i64, i64, i64, i64, vp, vp, vp, vp, vp, vp, ci, ci, vp]
            f.restype = ci
        for name in ("ref_matmul_f32", "ref_matmul_f64"):
            f = getattr(_lib, name)
            f.argtypes = [i64, i64, i64, vp, vp, vp, ci, ci, vp]
            f.restype = ci
        _lib.ref_matvec_f64.argtypes = [i64, i64, vp, vp, vp, ci, vp]
        _lib.ref_spmv_transfer_probe.argtypes = [vp]
    return _lib


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def _csr_call(entry, nrows, ncols, k, kout, rowptr, colind, values, x, w, out, reps, threads):
    times = np.zeros(max(reps, 1))
    rc = getattr(lib(), entry)(nrows, ncols, k, kout, _p(rowptr), _p(colind), _p(values), _p(x),
                               _p(w), _p(out), reps, threads, _p(times))
    if rc != 0:
        raise RuntimeError(f"{entry} failed ({rc})")
    return out, times[:reps]


def spmv_csr(rowptr, colind, values, x, reps=1, threads=1):
    """Emitted spmv (reference fixture tests/fixtures/spmv.mlir for int64 colind,
    oracle/ir/spmv_i32.mlir for int32 colind) on the serial stub."""
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    colind = np.ascontiguousarray(colind)
    values = np.ascontiguousarray(values, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    n = rowptr.shape[0] - 1
    entry = "ref_spmv_f64_i64" if colind.dtype == np.int64 else "ref_spmv_f64_i32"
    if colind.dtype not in (np.int64, np.int32):
        raise TypeError("colind must be int32 or int64")
    return _csr_call(entry, n, x.shape[0], 0, 0, rowptr, colind, values, x, None,
                     np.zeros(n), reps, threads)


def spmm_csr(rowptr, colind, values, X, reps=1, threads=1):
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    colind = np.ascontiguousarray(colind, dtype=np.int32)
    values = np.ascontiguousarray(values, dtype=np.float64)
    X = np.ascontiguousarray(X, dtype=np.float64)
    n = rowptr.shape[0] - 1
    return _csr_call("ref_spmm_f64_i32", n, X.shape[0], X.shape[1], 0, rowptr, colind, values,
                     X, None, np.zeros((n, X.shape[1])), reps, threads)


def gcn(rowptr, colind, values, X, W, reps=1, threads=1):
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    colind = np.ascontiguousarray(colind, dtype=np.int32)
    values = np.ascontiguousarray(values, dtype=np.float32)
    X = np.ascontiguousarray(X, dtype=np.float32)
    W = np.ascontiguousarray(W, dtype=np.float32)
    n = rowptr.shape[0] - 1
    return _csr_call("ref_gcn_f32_i32", n, X.shape[0], X.shape[1], W.shape[1], rowptr, colind,
                     values, X, W, np.zeros((n, W.shape[1]), dtype=np.float32), reps, threads)


def matmul(A, B, reps=1, threads=1):
    A = np.ascontiguousarray(A)
    B = np.ascontiguousarray(B, dtype=A.dtype)
    m, k = A.shape
    n = B.shape[1]
    out = np.zeros((m, n), dtype=A.dtype)
    entry = {np.dtype(np.float32): "ref_matmul_f32", np.dtype(np.float64): "ref_matmul_f64"}[A.dtype]
    times = np.zeros(max(reps, 1))
    rc = getattr(lib(), entry)(m, n, k, _p(A), _p(B), _p(out), reps, threads, _p(times))
    if rc != 0:
        raise RuntimeError(f"{entry} failed ({rc})")
    return out, times[:reps]


def matvec(A, x, reps=1):
    A = np.ascontiguousarray(A, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros(A.shape[0])
    times = np.zeros(max(reps, 1))
    lib().ref_matvec_f64(A.shape[0], A.shape[1], _p(A), _p(x), _p(y), reps, _p(times))
    return y, times[:reps]


def spmv_transfer_probe():
    """h2d_count, d2h_count, h2d_bytes, d2h_bytes of one emitted spmv call on the
    4x4 fixture (spmv_driver.cpp:43-50)."""
    out = np.zeros(4, dtype=np.int64)
    lib().ref_spmv_transfer_probe(_p(out))
    return tuple(int(v) for v in out)
