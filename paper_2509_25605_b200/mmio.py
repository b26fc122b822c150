"""On-disk sparse inputs: Matrix Market files -> CSR.

The paper's SpMV study runs SuiteSparse matrices, which ship
as Matrix Market coordinate files; the reference reads only its own args
format (`shape: / data: / file:` lines, tensors.py:25-104 — use
`lapis.tensors.load_args_file` for that, it feeds `runtime.run` unchanged).
`read_matrix_market` parses the file in the native library (parallel,
symmetric storage expanded, rows column-sorted) into numpy CSR arrays in the
layout the B200 kernels stream; `to_device` moves them to the GPU.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from . import _capi

SYMMETRY = {0: "general", 1: "symmetric", 2: "skew-symmetric", 3: "hermitian"}


def matrix_market_info(path) -> dict:
    out = (C.c_int64 * 4)()
    _capi.check(_capi.lib().lapis_b200_mm_info(str(path).encode(), out), "mm_info")
    return {"nrows": int(out[0]), "ncols": int(out[1]), "nnz": int(out[2]),
            "field": "pattern" if out[3] & 1 else ("integer" if out[3] & 2 else "real"),
            "symmetry": SYMMETRY[(out[3] >> 2) & 3]}


def read_matrix_market(path, index_dtype=np.int32, values: bool = True):
    """(rowptr int64, colind int32|int64, values f64 | None, (nrows, ncols))."""
    path = Path(path)
    info = matrix_market_info(path)
    rowptr = np.empty(info["nrows"] + 1, dtype=np.int64)
    colind = np.empty(info["nnz"], dtype=index_dtype)
    vals = np.empty(info["nnz"], dtype=np.float64) if values else None
    _capi.check(_capi.lib().lapis_b200_mm_read_csr(
        str(path).encode(), rowptr.ctypes.data_as(C.POINTER(C.c_int64)),
        C.c_void_p(colind.ctypes.data), colind.itemsize,
        vals.ctypes.data_as(C.POINTER(C.c_double)) if vals is not None else None),
        "mm_read_csr")
    return rowptr, colind, vals, (info["nrows"], info["ncols"])


def to_device(rowptr, colind, values, device="cuda"):
    import torch
    return tuple(torch.from_numpy(np.ascontiguousarray(a)).to(device) if a is not None else None
                 for a in (rowptr, colind, values))
