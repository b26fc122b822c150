"""Drop-in parity of the B200 executor (paper_2509_25605_b200.runtime.run)
against the reference interpreter (lapis.interp.run) on every reference
fixture program and every hot-path program of oracle/ir, lowered by the
reference pipeline and unlowered (golden files: tests/golden/make_run_golden.py).

Checked per case, as the reference's own tests check interp.run
(test_acceptance.py:183-270, test_interp.py:244-252):
* outputs — generated kernels (library=False) bit-identical; hand-written
  kernels bit-identical for integers, within diff_outputs tolerance for
  floats (1e-12 f64, 1e-5 f32: interp.py:1050-1071);
* the transfer trace (H2D / D2H bytes, SyncNoop, StaleAccess) — identical;
* the counters (single / barrier / store / hint per op path) — identical;
* the eager baseline's trace — identical.
"""
import numpy as np
import pytest

from conftest import bits_equal, load_run_case, run_cases

pytestmark = pytest.mark.gpu

lapis_parser = pytest.importorskip("lapis.parser")
from lapis.interp import diff_outputs, format_trace  # noqa: E402

CASES = run_cases()


def _tol(outputs) -> float:
    kinds = {np.asarray(o).dtype for o in outputs}
    return 1e-5 if np.dtype(np.float32) in kinds else 1e-12


def _run(text, case, **kw):
    from paper_2509_25605_b200 import runtime
    program = lapis_parser.parse(text)
    return runtime.run(program, case["entry"], [np.array(a, copy=True) for a in case["inputs"]], **kw)


@pytest.mark.parametrize("case_id", CASES)
def test_generated_bit_exact(case_id, cuda_device):
    case = load_run_case(case_id)
    r = _run(case["lowered"], case, library=False)
    assert len(r.outputs) == len(case["outputs"])
    for got, want in zip(r.outputs, case["outputs"]):
        assert bits_equal(np.asarray(got), want), (got, want)
    assert format_trace(r.trace) == case["trace"]
    assert {k: dict(v) for k, v in r.counters.items()} == case["counters"]


@pytest.mark.parametrize("case_id", CASES)
def test_library_kernels(case_id, cuda_device):
    case = load_run_case(case_id)
    r = _run(case["lowered"], case)
    rep = diff_outputs(r.outputs, case["outputs"], rel_tol=_tol(case["outputs"]))
    assert rep.match, str(rep)
    for got, want in zip(r.outputs, case["outputs"]):
        if np.asarray(want).dtype.kind in "iub":
            assert bits_equal(np.asarray(got), want)
    assert format_trace(r.trace) == case["trace"]
    assert {k: dict(v) for k, v in r.counters.items()} == case["counters"]


@pytest.mark.parametrize("case_id", CASES)
def test_exact_mode_bit_exact(case_id, cuda_device):
    case = load_run_case(case_id)
    r = _run(case["lowered"], case, exact=True)
    for got, want in zip(r.outputs, case["outputs"]):
        assert bits_equal(np.asarray(got), want)


@pytest.mark.parametrize("case_id", CASES)
def test_eager_trace(case_id, cuda_device):
    from paper_2509_25605_b200 import runtime
    case = load_run_case(case_id)
    program = lapis_parser.parse(case["lowered"])
    r = runtime.run_eager_baseline(program, case["entry"],
                                   [np.array(a, copy=True) for a in case["inputs"]])
    assert format_trace(r.trace) == case["eager_trace"]
    rep = diff_outputs(r.outputs, case["outputs"], rel_tol=_tol(case["outputs"]))
    assert rep.match, str(rep)


@pytest.mark.parametrize("case_id", CASES)
def test_unlowered_program(case_id, cuda_device):
    case = load_run_case(case_id)
    r = _run(case["orig"], case)
    rep = diff_outputs(r.outputs, case["orig_outputs"], rel_tol=_tol(case["orig_outputs"]))
    assert rep.match, str(rep)
    assert format_trace(r.trace) == case["orig_trace"]
    assert {k: dict(v) for k, v in r.counters.items()} == case["orig_counters"]


HOT = {"spmv": "spmv", "spmv_loops": "spmv", "ir_spmv_i32": "spmv", "ir_spmm": "spmm",
       "matmul_f64": "gemm", "matmul_i32": "gemm", "ir_matmul_f32": "gemm", "ir_matmul_f64": "gemm",
       "matvec_f64": "gemv", "ir_matvec_f64": "gemv", "axis_reduce": "reduce", "depth2": "reduce",
       "ir_gcn_f32": "spmm+gemm+relu"}


@pytest.mark.parametrize("name", sorted(HOT))
def test_hot_nests_run_hand_written_kernels(name, cuda_device):
    """The hot nests of the lowered programs take the hand-written kernels
    (no silent generated-kernel path for them)."""
    case = load_run_case(f"{name}.b")
    r = _run(case["lowered"], case)
    assert r.kernels and all(kind == "library" for _, kind in r.kernels), r.kernels
