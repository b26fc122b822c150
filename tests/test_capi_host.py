"""CPU-side checks of the boundary: the library loads, exports every symbol
include/lapis_b200.h declares, host-only entries answer correctly, and the
product path refuses to run without a GPU (no CPU fallback)."""
import re
from pathlib import Path

import pytest
import torch

import paper_2509_25605_b200 as lb
from paper_2509_25605_b200 import _capi
from oracle import oracle as O

HEADER = Path(__file__).resolve().parent.parent / "include" / "lapis_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(lapis_b200_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _capi.lib()
    syms = declared_symbols()
    assert len(syms) >= 15
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(_capi._SIGNATURES), "ctypes signatures out of sync with the header"


def test_version_and_error_channel():
    assert _capi.lib().lapis_b200_version() >= 100
    assert isinstance(_capi.last_error(), str)


@pytest.mark.parametrize("nrows,nnz,cap", [(4, 5, 32), (300, 4302, 32), (1_000_000, 4_996_000, 32),
                                           (10_000_000, 99_891_811, 32), (64, 4096, 16), (0, 0, 32),
                                           (7, 1000, 8), (200_201_625, 5_386_984_777, 32)])
def test_vector_length_rule_matches_oracle(nrows, nnz, cap):
    assert lb.csr_vector_length(nrows, nnz, cap) == O.csr_vector_length(nrows, nnz, cap)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    rowptr = torch.tensor([0, 1], dtype=torch.int64)
    with pytest.raises(lb.BackendError):
        lb.spmv_csr(rowptr, torch.tensor([0]), torch.tensor([1.0]), torch.tensor([1.0]))
    with pytest.raises(lb.BackendError):
        lb.gemm(torch.ones(2, 2), torch.ones(2, 2))
