"""CPU checks of the generated-kernel path: every device nest and library op
of every drop-in case (tests/golden/run, lowered and original programs)
generates CUDA that NVRTC compiles for sm_100a (no device needed)."""
import ctypes as C

import pytest

from conftest import RUN_GOLDEN, load_run_case, run_cases

lapis_parser = pytest.importorskip("lapis.parser")

from paper_2509_25605_b200 import _capi, cudagen  # noqa: E402

NAMES = sorted({p.name.split(".")[0] for p in RUN_GOLDEN.glob("*.mlir")})


def _kernel_roots(program):
    from lapis.ir import walk
    out = []
    for func in program.funcs():
        for op in walk(func):
            if op.name in cudagen.LIBRARY_OPS:
                out.append(op)
            elif op.name in ("kokkos.range_parallel", "kokkos.thread_parallel",
                             "kokkos.team_parallel") and op.attrs.get("executionSpace") == "device":
                out.append(op)
            elif op.name == "scf.parallel" and not any(
                    a.name in ("scf.parallel", "kokkos.range_parallel") for a in op.ancestors()):
                out.append(op)
    return out


def _check(src: str, name: str) -> int:
    n = C.c_int64()
    rc = _capi.lib().lapis_b200_jit_check(src.encode(), name.encode(), C.byref(n))
    assert rc == 0, _capi.last_error() + "\n" + src
    return n.value


@pytest.mark.skipif(not _capi.lib().lapis_b200_jit_available(), reason="NVRTC not loadable")
@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("form", ["lowered", "orig"])
def test_generated_kernels_compile(name, form):
    program = lapis_parser.parse((RUN_GOLDEN / f"{name}.{form}.mlir").read_text())
    roots = _kernel_roots(program)
    from lapis.ir import walk
    for i, op in enumerate(roots):
        if any(o.name == "memref.alloc" for o in walk(op)):
            continue  # per-iteration allocations stay host code (runtime._device_mappable)
        for vl in (1, 8):
            kname = f"k{i}_{vl}"
            if op.name in cudagen.LIBRARY_OPS:
                k = cudagen.generate_library(op, kname)
            else:
                k = cudagen.generate(op, kname, vl=vl)
            assert _check(k.source, k.name) > 0
            if k.fold_name:
                assert _check(k.source, k.fold_name) > 0


@pytest.mark.parametrize("case_id", run_cases())
def test_run_golden_cases_load(case_id):
    case = load_run_case(case_id)
    assert case["outputs"] and case["entry"]
    program = lapis_parser.parse(case["lowered"])
    assert program.find_func(case["entry"]) is not None
