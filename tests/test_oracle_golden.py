"""Pin the oracle (oracle/lapis_oracle.c) to the reference's own outputs.

Every fixture under tests/golden/ was produced by the reference interpreter
(tests/golden/make_golden.py).  The C restatement must reproduce each one
bit for bit — floats included — because it follows the same sequential,
per-op-rounded order (interp.py:168-183, 711-812).
"""
import numpy as np
import pytest

from conftest import bits_equal, golden_names, load_golden
from oracle import oracle as O


@pytest.mark.parametrize("name", golden_names("spmv"))
def test_spmv_bitexact(name):
    g = load_golden(name)
    rowptr, colind, values, x, _ = g["inputs"]
    y = O.spmv_csr(rowptr, colind, values, x)
    assert bits_equal(y, g["outputs"][0]), name
    assert bits_equal(g["orig"][0], g["outputs"][0])  # the pipeline preserved semantics


@pytest.mark.parametrize("name", golden_names("spmv"))
def test_vector_length_hint(name):
    g = load_golden(name)
    rowptr = g["inputs"][0]
    n = rowptr.shape[0] - 1
    assert O.csr_vector_length(n, int(rowptr[-1]) if n >= 0 else 0) == g["hints"][0]


def test_hint_formula_table():
    # test_loop_mapping.py:150-180 / test_acceptance.py:194-205 and SURVEY A.10
    assert O.csr_vector_length(4, 5) == 2
    assert O.csr_vector_length(300, 4302) == 16
    assert O.csr_vector_length(1_000_000, 4_996_000) == 8        # config 1
    assert O.csr_vector_length(10_000_000, 99_891_811) == 16     # config 3
    assert O.csr_vector_length(200_201_625, 5_386_984_777) == 32  # config 5
    assert O.csr_vector_length(64, 64 * 64, cap=16) == 16
    assert O.csr_vector_length(0, 0) == 1


@pytest.mark.parametrize("name", ["matmul_i32", "matmul_f64", "matmul_f64_kl",
                                  "matmul_dyn_f32", "matmul_dyn_f64"])
def test_matmul_bitexact(name):
    g = load_golden(name)
    A, B = g["inputs"][:2]
    assert bits_equal(O.matmul(A, B), g["outputs"][0])


def test_matmul_entries_match_full():
    g = load_golden("matmul_dyn_f32")
    A, B = g["inputs"][:2]
    ii = np.array([0, 3, 44, 20]); jj = np.array([0, 69, 5, 33])
    assert bits_equal(O.matmul_entries(A, B, ii, jj), g["outputs"][0][ii, jj])


@pytest.mark.parametrize("name", ["matvec_f64", "matvec_f64_kl", "matvec_dyn"])
def test_matvec_bitexact(name):
    g = load_golden(name)
    A, x = g["inputs"][:2]
    assert bits_equal(O.matvec(A, x), g["outputs"][0])


def test_batch_matmul_bitexact():
    g = load_golden("batch_matmul_f32")
    A, B = g["inputs"]
    assert bits_equal(O.batch_matmul(A, B), g["outputs"][0])


@pytest.mark.parametrize("name", golden_names("reduce_"))
def test_reduce_bitexact(name):
    g = load_golden(name)
    if name == "reduce_add_f64":
        src, out = g["inputs"][0], g["outputs"][0]
        assert bits_equal(O.reduce2d(src, 1, "add"), out)
        return
    _, comb, ax, _ = name.split("_")
    assert bits_equal(O.reduce2d(g["inputs"][0], int(ax[2:]), comb), g["outputs"][0])


def test_spmm_bitexact():
    g = load_golden("spmm_k8")
    rowptr, colind, values, X, _ = g["inputs"]
    assert bits_equal(O.spmm_csr(rowptr, colind, values, X), g["outputs"][0])


def test_gcn_bitexact():
    g = load_golden("gcn_small")
    rowptr, colind, values, X, W, _ = g["inputs"]
    assert bits_equal(O.gcn(rowptr, colind, values, X, W), g["outputs"][0])


def test_row_range_and_threads_do_not_change_bits():
    g = load_golden("spmv_ragged400")
    rowptr, colind, values, x, _ = g["inputs"]
    full = g["outputs"][0]
    part = O.spmv_csr(rowptr, colind, values, x, rows=(100, 250), threads=3)
    assert bits_equal(part[100:250], full[100:250])
    assert not part[:100].any() and not part[250:].any()
