"""Generate tests/golden/run/ — drop-in parity cases for ``runtime.run`` — from
the REFERENCE ITSELF.

Run in the build container (the reference is importable there; the GPU box
only reads the committed files):

    python tests/golden/make_run_golden.py

For every reference fixture program (the reference suite's
``tests/fixtures/*.mlir``) and every hot-path program under ``oracle/ir/``:

* ``<name>.lowered.mlir`` — the program after the reference's preset pipeline
  (``run_pipeline(..., PassPipeline.preset(), TargetConfig())``), printed by
  the reference printer;
* ``<name>.orig.mlir`` — the unlowered program, printed by the reference
  printer (parse -> print normalisation);
* ``<name>.npz`` — seeded inputs (the reference suite's own generators,
  ``conftest.random_inputs`` / ``spmv4_inputs`` / ``random_csr``) and, from
  the reference interpreter ``lapis.interp.run``: the outputs of the lowered
  and of the original program, the lazy trace, the eager trace and the
  counters, JSON-encoded.
"""
from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("LAPIS_REFERENCE", "/root/reference")) / "pkg"
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))

from lapis.interp import format_trace, run, run_eager_baseline  # noqa: E402
from lapis.parser import parse_file  # noqa: E402
from lapis.passes import PassPipeline, TargetConfig, run_pipeline  # noqa: E402
from lapis.printer import print_program  # noqa: E402

import conftest as refc  # noqa: E402

HERE = Path(__file__).resolve().parent
OUT = HERE / "run"
IR = HERE.parent.parent / "oracle" / "ir"


def case_inputs(name, program, rng):
    if name in ("spmv", "spmv_loops"):
        if rng is None:
            return refc.spmv4_inputs()
        rowptr, colind, values, _ = refc.random_csr(rng, 60, 50, 0.2)
        return [rowptr, colind, values, rng.uniform(-1, 1, 50), np.zeros(60)]
    if name in ("ir_spmm", "ir_spmv_i32", "ir_gcn_f32"):
        g = rng or np.random.default_rng(7)
        rows, cols, k = 40, 40, 8
        rowptr, colind, values, _ = refc.random_csr(g, rows, cols, 0.15)
        if name == "ir_spmv_i32":
            return [rowptr.astype(np.int32), colind.astype(np.int32), values,
                    g.uniform(-1, 1, cols), np.zeros(rows)]
        ci32 = colind.astype(np.int32)
        if name == "ir_spmm":
            return [rowptr, ci32, values, g.uniform(-1, 1, (cols, k)), np.zeros((rows, k))]
        return [rowptr, ci32, np.abs(values).astype(np.float32),
                g.uniform(0, 1, (cols, k)).astype(np.float32),
                g.uniform(-0.125, 0.125, (k, k)).astype(np.float32),
                np.zeros((rows, k), dtype=np.float32)]
    return refc.random_inputs(program, rng or np.random.default_rng(11))


def encode_counters(c: dict) -> str:
    return json.dumps({k: dict(v) for k, v in c.items()}, sort_keys=True)


def main() -> None:
    OUT.mkdir(exist_ok=True)
    sources = [(p.stem, p) for p in sorted((REF / "tests" / "fixtures").glob("*.mlir"))]
    sources += [("ir_" + p.stem, p) for p in sorted(IR.glob("*.mlir"))]
    # the kernel-library route (kokkos.gemm / gemv -> LAPIS::gemm / gemv) of the dense programs
    kl = [("kl_" + n, p) for n, p in sources if n in ("matmul_f64", "matmul_i32", "matvec_f64",
                                                      "ir_matmul_f32", "ir_matmul_f64",
                                                      "ir_matvec_f64")]
    for name, path in sources + kl:
        program = parse_file(str(path))
        cfg = TargetConfig(kernel_library_calls=True) if name.startswith("kl_") else TargetConfig()
        lowered = run_pipeline(program, PassPipeline.preset(), cfg).program
        entry = program.funcs()[0].attrs["sym_name"]
        (OUT / f"{name}.lowered.mlir").write_text(print_program(lowered))
        (OUT / f"{name}.orig.mlir").write_text(print_program(program))
        for seed_tag, rng in (("a", None), ("b", np.random.default_rng(1234))):
            inputs = case_inputs(name, program, rng)
            lazy = run(lowered, entry, [np.array(a, copy=True) for a in inputs])
            eager = run_eager_baseline(lowered, entry, [np.array(a, copy=True) for a in inputs])
            orig = run(program, entry, [np.array(a, copy=True) for a in inputs])
            arrays = {f"in{i}": np.asarray(a) for i, a in enumerate(inputs)}
            arrays.update({f"out{i}": np.asarray(a) for i, a in enumerate(lazy.outputs)})
            arrays.update({f"orig{i}": np.asarray(a) for i, a in enumerate(orig.outputs)})
            arrays["entry"] = np.array(entry)
            arrays["trace"] = np.array(format_trace(lazy.trace))
            arrays["eager_trace"] = np.array(format_trace(eager.trace))
            arrays["orig_trace"] = np.array(format_trace(orig.trace))
            arrays["counters"] = np.array(encode_counters(lazy.counters))
            arrays["orig_counters"] = np.array(encode_counters(orig.counters))
            np.savez(OUT / f"{name}.{seed_tag}.npz", **arrays)
        print(name)


if __name__ == "__main__":
    main()
