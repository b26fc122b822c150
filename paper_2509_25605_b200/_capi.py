"""ctypes binding of the C ABI in include/lapis_b200.h.

The shared library is built in-tree (paper_2509_25605_b200/build.py) and
loaded from ``paper_2509_25605_b200/lib/liblapis_b200.so``.  There is no CPU
fallback: if the library is missing or no CUDA device is present, every call
raises :class:`BackendError`.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "lib" / "liblapis_b200.so"

OK, ERR_ARG, ERR_CUDA, ERR_UNSUPPORTED, ERR_NOMEM = 0, 1, 2, 3, 4
F32, F64, I32, I64 = 0, 1, 2, 3
ADD, MUL, MIN, MAX = 0, 1, 2, 3
GEMM_AUTO, GEMM_TF32X3, GEMM_DMMA, GEMM_EXACT, GEMM_OZAKI = 0, 1, 2, 3, 4


class BackendError(RuntimeError):
    """Raised for every nonzero status; carries the library's last_error text.

    Mirrors the reference's InterpError shape (a message plus an optional
    location, interp.py:40-43) so callers can treat both alike."""

    def __init__(self, message: str, code: int = ERR_CUDA, path: str = ""):
        super().__init__(message + (f" at {path}" if path else ""))
        self.code = code
        self.path = path


_lib: C.CDLL | None = None

_I64, _VP, _INT = C.c_int64, C.c_void_p, C.c_int
_SIGNATURES = {
    "lapis_b200_last_error": ([], C.c_char_p),
    "lapis_b200_version": ([], _INT),
    "lapis_b200_init": ([_INT], _INT),
    "lapis_b200_nccl_unique_id": ([_VP], _INT),
    "lapis_b200_nccl_comm_init": ([_VP, _INT, _INT, _VP], _INT),
    "lapis_b200_nccl_comm_destroy": ([_VP], _INT),
    "lapis_b200_rowblock_create": ([_VP, _INT, _INT, _VP, _VP, _INT, _VP, _INT, _I64, _INT, _VP,
                                    _VP], _INT),
    "lapis_b200_rowblock_info": ([_VP, _VP], _INT),
    "lapis_b200_spmv_csr_rowblock": ([_VP, _VP, _INT, _VP, _INT, _VP, _VP, _VP, _INT, _VP], _INT),
    "lapis_b200_rowblock_destroy": ([_VP], _INT),
    "lapis_b200_finalize": ([], _INT),
    "lapis_b200_csr_vector_length": ([_I64, _I64, _I64], _I64),
    "lapis_b200_spmv_csr": ([_I64, _I64, _I64, _VP, _INT, _VP, _INT, _VP, _VP, _VP, _INT, _INT,
                             _VP], _INT),
    "lapis_b200_csr_plan_create": ([_I64, _I64, _VP, _INT, _VP, C.POINTER(_VP)], _INT),
    "lapis_b200_csr_plan_destroy": ([_VP], _INT),
    "lapis_b200_spmv_csr_plan": ([_VP, _VP, _INT, _VP, _INT, _VP, _VP, _VP, _INT, _VP], _INT),
    "lapis_b200_csr_plan_info": ([_VP, _VP], _INT),
    "lapis_b200_csr_plan_set_exact": ([_VP, _INT], _INT),
    "lapis_b200_spmm_csr": ([_I64, _I64, _I64, _I64, _VP, _INT, _VP, _INT, _VP, _VP, _I64, _VP,
                             _I64, _INT, _VP], _INT),
    "lapis_b200_gemm": ([_I64, _I64, _I64, _VP, _I64, _VP, _I64, _VP, _I64, _INT, _INT, _VP], _INT),
    "lapis_b200_gemv": ([_I64, _I64, _VP, _I64, _VP, _VP, _INT, _VP], _INT),
    "lapis_b200_batch_gemm": ([_I64, _I64, _I64, _I64, _VP, _VP, _VP, _INT, _INT, _VP], _INT),
    "lapis_b200_reduce_2d": ([_I64, _I64, _VP, _VP, _INT, _INT, _INT, _VP], _INT),
    "lapis_b200_relu": ([_I64, _VP, _VP, _INT, _VP], _INT),
    "lapis_b200_gcn_layer": ([_I64, _I64, _I64, _VP, _INT, _VP, _INT, _VP, _VP, _I64, _VP, _I64,
                              _VP, _INT, _VP], _INT),
    "lapis_b200_spmm_plan_create": ([_I64, _I64, _I64, _I64, _VP, _INT, _VP, _INT, _INT, _I64, _VP,
                                     C.POINTER(_VP)], _INT),
    "lapis_b200_spmm_plan_info": ([_VP, C.POINTER(_I64)], _INT),
    "lapis_b200_spmm_plan_hints": ([_VP, C.POINTER(_I64)], _INT),
    "lapis_b200_spmm_plan_destroy": ([_VP], _INT),
    "lapis_b200_spmm_csr_plan": ([_VP, _VP, _INT, _VP, _INT, _VP, _VP, _I64, _VP, _I64, _INT, _VP],
                                 _INT),
    "lapis_b200_graph_kernels": ([_VP, C.c_char_p, _I64, C.POINTER(_I64)], _INT),
    "lapis_b200_gcn_layer_mode": ([_I64, _I64, _I64, _VP, _INT, _VP, _INT, _VP, _VP, _I64, _VP,
                                   _I64, _VP, _INT, _INT, _VP], _INT),
    "lapis_b200_synth_stencil": ([_INT, _I64, _I64, _I64, _VP, _VP, _VP, _VP], _INT),
    "lapis_b200_csr_check": ([_I64, _VP, _INT, _VP, _INT, _I64, _I64, C.POINTER(_I64), _VP],
                             _INT),
    "lapis_b200_mm_info": ([C.c_char_p, C.POINTER(_I64)], _INT),
    "lapis_b200_mm_read_csr": ([C.c_char_p, C.POINTER(_I64), _VP, _INT, C.POINTER(C.c_double)],
                               _INT),
    "lapis_b200_jit_available": ([], _INT),
    "lapis_b200_jit_compile": ([C.c_char_p, C.c_char_p, C.POINTER(_VP)], _INT),
    "lapis_b200_jit_launch": ([_VP, _I64, _INT, _INT, _VP, _I64, _VP], _INT),
    "lapis_b200_jit_cache_size": ([], _INT),
    "lapis_b200_jit_check": ([C.c_char_p, C.c_char_p, C.POINTER(_I64)], _INT),
}


def library_path() -> Path:
    return LIB_PATH


def lib() -> C.CDLL:
    """Load the backend library (raises BackendError if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise BackendError(f"CUDA backend not built: {LIB_PATH} is missing "
                               "(run __graft_entry__.build())", ERR_UNSUPPORTED)
        handle = C.CDLL(str(LIB_PATH))
        for name, (args, res) in _SIGNATURES.items():
            f = getattr(handle, name)
            f.argtypes = args
            f.restype = res
        _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().lapis_b200_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    if rc != OK:
        raise BackendError(f"{what}: {last_error()}" if what else last_error(), rc)
