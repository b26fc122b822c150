"""The kernel-library route for CSR SpMV (paper_2509_25605_b200.sparse_route,
SURVEY §8f-1): `sparse.spmv_csr` -> `kokkos.spmv_csr` -> `LAPIS::spmv_csr(...)`.

CPU: the reference pipeline with kernel_library_calls rewrites the op (and
leaves the default pipeline byte-identical to the golden lowering); the
reference interpreter runs the routed program with the same outputs (bit for
bit: same arithmetic) and the same transfer trace as the loop route; the
reference emitter writes the library call.  GPU: runtime.run executes the
routed op on the tuned kernels, and the emitted C++ compiled for sm_100a binds
LAPIS::spmv_csr to lapis_b200_spmv_csr."""
import re
import subprocess

import numpy as np
import pytest

import cxx_drivers as D
from conftest import bits_equal, load_run_case

lapis_parser = pytest.importorskip("lapis.parser")
from lapis import interp  # noqa: E402
from lapis.interp import diff_outputs, format_trace  # noqa: E402
from lapis.passes import PassPipeline, TargetConfig, run_pipeline  # noqa: E402

from paper_2509_25605_b200 import sparse_route  # noqa: E402

sparse_route.install()
CASES = ["spmv.a", "spmv.b", "ir_spmv_i32.a", "ir_spmv_i32.b"]


def _lower(text, routed=True):
    program = lapis_parser.parse(text)
    cfg = TargetConfig(kernel_library_calls=routed)
    return run_pipeline(program, PassPipeline.preset(), cfg).program


def _inputs(case):
    return [np.array(a, copy=True) for a in case["inputs"]]


@pytest.mark.parametrize("case_id", CASES)
def test_route_rewrites_spmv(case_id):
    from lapis.printer import print_program
    case = load_run_case(case_id)
    text = print_program(_lower(case["orig"]))
    assert "kokkos.spmv_csr" in text and "sparse.spmv_csr" not in text
    assert "kokkos.sync" in text and "kokkos.modify" in text          # DualView management
    # the default pipeline is untouched by the installed pass
    assert print_program(_lower(case["orig"], routed=False)).strip() == case["lowered"].strip()


@pytest.mark.parametrize("case_id", CASES)
def test_routed_interp_matches_loop_route(case_id):
    case = load_run_case(case_id)
    program = _lower(case["orig"])
    r = interp.run(program, case["entry"], _inputs(case))
    for got, want in zip(r.outputs, case["outputs"]):
        assert bits_equal(np.asarray(got), want)
    ours = [t for t in format_trace(r.trace).splitlines() if t.startswith(("H2D", "D2H"))]
    loop = [t for t in case["trace"].splitlines() if t.startswith(("H2D", "D2H"))]
    assert sorted(ours) == sorted(loop)       # same transfers (the op syncs in operand order)
    eager = interp.run_eager_baseline(program, case["entry"], _inputs(case))
    for got, want in zip(eager.outputs, case["outputs"]):
        assert bits_equal(np.asarray(got), want)
    assert sum(1 for t in format_trace(eager.trace).splitlines() if t.startswith("H2D")) >= 4


def test_routed_emitter_writes_library_call():
    from lapis.emitter import EmitOptions, emit
    case = load_run_case("spmv.a")
    src = emit(_lower(case["orig"]), EmitOptions(header_name="kl_spmv")).source
    assert re.search(r"LAPIS::spmv_csr\(\w+, \w+, \w+, \w+, \w+\);", src)


def test_unrouted_default_has_no_library_call():
    from lapis.emitter import EmitOptions, emit
    case = load_run_case("spmv.a")
    src = emit(_lower(case["orig"], routed=False), EmitOptions(header_name="spmv")).source
    assert "LAPIS::spmv_csr" not in src


@pytest.mark.skipif(D.nvcc() is None or not D.emitted_cases(), reason="no nvcc / runtime header")
def test_emitted_routed_cpp_compiles_for_sm100a(tmp_path):
    name, program, case, src = _emit_driver("spmv.b", tmp_path)
    r = D.compile_driver(src, tmp_path / f"{name}.o", compile_only=True, b200_seam=True,
                         extra_include=tmp_path)
    assert r.returncode == 0, r.stderr[-3000:]


def _emit_driver(case_id, d):
    from lapis.emitter import EmitOptions, emit
    from lapis.runtime_header import RUNTIME_HEADER_NAME, emit_runtime_header
    case = load_run_case(case_id)
    program = _lower(case["orig"])
    name = "kl_" + case_id.split(".")[0]
    (d / f"{name}.hpp").write_text(emit(program, EmitOptions(header_name=name)).source)
    (d / RUNTIME_HEADER_NAME).write_text(emit_runtime_header())
    inputs = D.coerce_inputs(program, case["entry"], case["inputs"])
    src = d / f"{name}.cu"
    src.write_text(D.driver_source(name, program, case["entry"], inputs, b200_seam=True))
    D.write_inputs(d, inputs)
    return name, program, case, src


# ----------------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("case_id", CASES)
def test_runtime_runs_routed_program(case_id, cuda_device):
    from paper_2509_25605_b200 import runtime
    case = load_run_case(case_id)
    program = _lower(case["orig"])
    want = interp.run(program, case["entry"], _inputs(case))
    for exact in (False, True):
        r = runtime.run(program, case["entry"], _inputs(case), exact=exact)
        rep = diff_outputs(r.outputs, want.outputs, rel_tol=1e-12)
        assert rep.match, str(rep)
        if exact:
            for got, w in zip(r.outputs, want.outputs):
                assert bits_equal(np.asarray(got), np.asarray(w))
        assert format_trace(r.trace) == format_trace(want.trace)
        if not exact:   # the tuned kernel ran (exact mode may pick the generated one)
            assert [k for _, k in r.kernels] == ["library"], r.kernels


@pytest.mark.gpu
@pytest.mark.skipif(D.nvcc() is None, reason="no nvcc")
@pytest.mark.parametrize("case_id", ["spmv.b", "ir_spmv_i32.b"])
def test_emitted_routed_cpp_on_b200(case_id, cuda_device, tmp_path):
    name, program, case, src = _emit_driver(case_id, tmp_path)
    exe = tmp_path / name
    r = D.compile_driver(src, exe, b200_seam=True, extra_include=tmp_path)
    assert r.returncode == 0, r.stderr[-3000:]
    nm = subprocess.run(["nm", "-C", str(exe)], capture_output=True, text=True).stdout
    assert "lapis_b200_spmv_csr" in nm
    run = subprocess.run([str(exe), str(tmp_path)], capture_output=True, text=True, timeout=120)
    assert run.returncode == 0, run.stderr[-2000:]
    want = interp.run(program, case["entry"], _inputs(case))
    got = D.read_output(tmp_path, np.asarray(want.outputs[0]))
    rep = diff_outputs([got], [np.asarray(want.outputs[0])], rel_tol=1e-12)
    assert rep.match, str(rep)
    stats = dict(re.findall(r"(\w+)=(\d+)", run.stdout))
    trace = format_trace(want.trace).splitlines()
    assert int(stats["h2d_count"]) == sum(1 for t in trace if t.startswith("H2D"))
    assert int(stats["d2h_count"]) == sum(1 for t in trace if t.startswith("D2H"))
