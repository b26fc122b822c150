"""The reference-emitted Kokkos C++ on B200: every drop-in case's emitted
header (the reference CLI's `translate` of tests/golden/run/<name>.lowered.mlir,
built into oracle/_ref/emitted by __graft_entry__.build()) compiled UNCHANGED
with nvcc for sm_100a against include/kokkos_b200/Kokkos_Core.hpp, together
with the reference's own generated runtime header.

CPU: a few drivers compile (header regressions).  GPU: every driver compiles,
runs, and matches the reference interpreter's outputs (ints exact, floats
within diff_outputs tolerance: Kokkos vector / team reductions are trees) and
its transfer counts (LAPIS::transferStats vs the interpreter trace)."""
import concurrent.futures as cf
import re
import subprocess
import tempfile
from pathlib import Path

import numpy as np
import pytest

import cxx_drivers as D
from conftest import load_run_case

lapis_parser = pytest.importorskip("lapis.parser")

CASES = D.emitted_cases()
needs_build = pytest.mark.skipif(not CASES or D.nvcc() is None,
                                 reason="emitted C++ not built (oracle/_ref/emitted) or no nvcc")


def _seam(name: str) -> bool:
    # kernel-library route: LAPIS::gemm / gemv through include/lapis_b200_runtime.hpp
    return name.startswith("kl_")


def _prepare(name: str, d: Path):
    case = load_run_case(f"{name}.b")
    program = lapis_parser.parse(case["lowered"])
    src = d / f"{name}.cu"
    inputs = D.coerce_inputs(program, case["entry"], case["inputs"])
    src.write_text(D.driver_source(name, program, case["entry"], inputs, b200_seam=_seam(name)))
    D.write_inputs(d, inputs)
    return case, src


@needs_build
@pytest.mark.parametrize("name", [n for n in ("spmv", "team_single_barrier", "globals",
                                              "kl_matmul_f64") if n in CASES])
def test_emitted_cpp_compiles_for_sm100a(name, tmp_path):
    _, src = _prepare(name, tmp_path)
    r = D.compile_driver(src, tmp_path / f"{name}.o", compile_only=True, b200_seam=_seam(name))
    assert r.returncode == 0, r.stderr[-3000:]


@pytest.fixture(scope="module")
def built():
    """Compile every driver once (in parallel) on the GPU box."""
    root = Path(tempfile.mkdtemp(prefix="kokkos_b200_"))
    out = {}

    def one(name):
        d = root / name
        d.mkdir()
        case, src = _prepare(name, d)
        exe = d / "drv"
        r = D.compile_driver(src, exe, b200_seam=_seam(name))
        return name, (case, d, exe, r)

    with cf.ThreadPoolExecutor(8) as ex:
        for name, v in ex.map(one, CASES):
            out[name] = v
    return out


@pytest.mark.gpu
@needs_build
@pytest.mark.parametrize("name", CASES)
def test_emitted_cpp_runs_on_b200(name, built, cuda_device):
    from lapis.interp import diff_outputs
    case, d, exe, r = built[name]
    assert r.returncode == 0, r.stderr[-3000:]
    if _seam(name):
        # the emitted LAPIS::gemm / gemv bound to the B200 kernels, not the
        # runtime header's generic templates
        syms = subprocess.run(["nm", "-D", "--undefined-only", str(exe)], capture_output=True,
                              text=True).stdout
        assert "lapis_b200_gemm" in syms or "lapis_b200_gemv" in syms, syms[-500:]
    run = subprocess.run([str(exe), str(d)], capture_output=True, text=True, timeout=120)
    assert run.returncode == 0, run.stderr[-2000:]
    want = np.asarray(case["outputs"][0])
    got = D.read_output(d, want)
    tol = 1e-5 if want.dtype == np.float32 else 1e-12
    rep = diff_outputs([got], [want], rel_tol=tol)
    assert rep.match, str(rep)
    stats = dict(re.findall(r"(\w+)=(\d+)", run.stdout))
    trace = case["trace"].splitlines()
    assert int(stats["h2d_count"]) == sum(1 for t in trace if t.startswith("H2D"))
    assert int(stats["d2h_count"]) == sum(1 for t in trace if t.startswith("D2H"))
