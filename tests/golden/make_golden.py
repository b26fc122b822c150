"""Generate tests/golden/*.npz from the REFERENCE ITSELF.

Run in the build container (the reference is importable there; it is not on
the GPU box, which only reads the committed fixtures):

    python tests/golden/make_golden.py

Every fixture is produced by the reference interpreter (``lapis.interp.run``,
the reference's "semantic oracle") on the program lowered by the reference's
preset pipeline (``run_pipeline(..., PassPipeline.preset(), TargetConfig())``),
using the reference test suite's own input generators (``conftest.py``:
``spmv4_inputs``, ``random_csr``, ``csr_with_mean``, ``random_inputs``).  Each
npz holds the inputs ``in0..inN``, the lowered-program outputs ``out0..``, the
unlowered-program outputs ``orig0..``, the copy-event trace and the observed
vector-length hints.
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

from lapis.interp import copy_events, run  # noqa: E402
from lapis.parser import parse, parse_file  # noqa: E402
from lapis.passes import PassPipeline, TargetConfig, run_pipeline  # noqa: E402

import conftest as refc  # noqa: E402  (the reference test suite's generators)

HERE = Path(__file__).resolve().parent
IR = HERE.parent.parent / "oracle" / "ir"


def lower(program, **cfg):
    return run_pipeline(program, PassPipeline.preset(), TargetConfig(**cfg)).program


def spmv_text(rp="index", ci="index", vt="f64"):
    return f"""
    func @spmv(%rowptr: memref<?x{rp}>, %colind: memref<?x{ci}>, %values: memref<?x{vt}>,
               %x: memref<?x{vt}>, %y: memref<?x{vt}>) -> (memref<?x{vt}>) {{
      sparse.spmv_csr(%rowptr, %colind, %values, %x, %y)
      func.return(%y)
    }}
    """


def reduce_text(shape, vt, axes, comb):
    rows, cols = shape
    out = rows if axes == [1] else cols
    return f"""
    func @red(%a: memref<{rows}x{cols}x{vt}>) -> (memref<{out}x{vt}>) {{
      %out = memref.alloc() : memref<{out}x{vt}>
      linalg.reduce(%a, %out) {{axes = {axes}, combiner = {comb}}}
      func.return(%out)
    }}
    """


def save(name, original, entry, inputs, **cfg):
    lowered = lower(original, **cfg)
    res = run(lowered, entry, [np.copy(v) if isinstance(v, np.ndarray) else v for v in inputs])
    orig = run(original, entry, [np.copy(v) if isinstance(v, np.ndarray) else v for v in inputs])
    payload = {f"in{i}": np.asarray(v) for i, v in enumerate(inputs)}
    payload.update({f"out{i}": np.asarray(v) for i, v in enumerate(res.outputs)})
    payload.update({f"orig{i}": np.asarray(v) for i, v in enumerate(orig.outputs)})
    payload["trace"] = np.array(json.dumps([str(e) for e in copy_events(res.trace)]))
    payload["hints"] = np.array(json.dumps(list(res.counters["hint"].values())))
    np.savez_compressed(HERE / f"{name}.npz", **payload)
    print(f"{name}: outputs={[np.asarray(o).shape for o in res.outputs]} "
          f"hints={list(res.counters['hint'].values())} copies={len(copy_events(res.trace))}")


def main():
    spmv = parse_file(str(REF / "tests/fixtures/spmv.mlir"))
    # test_interp.py:19-28 / conftest.py:59-69 — the 4x4 KAT, y = [3, 3, 0, 9]
    save("spmv4", spmv, "spmv", refc.spmv4_inputs())
    # test_spmv_lowering.py:36-43 — identity
    save("spmv_identity", spmv, "spmv",
         [np.array([0, 1, 2, 3], dtype=np.int64), np.array([0, 1, 2], dtype=np.int64),
          np.ones(3), np.array([1.0, 2.0, 3.0]), np.zeros(3)])
    # test_spmv_lowering.py:46-53 (seed 31) and test_acceptance.py:85-97 (seed 77)
    for seed in (31, 77):
        rng = np.random.default_rng(seed)
        rowptr, colind, values, _ = refc.random_csr(rng, 100, 100, 0.05)
        x = rng.uniform(-1.0, 1.0, 100)
        save(f"spmv_random100_s{seed}", spmv, "spmv", [rowptr, colind, values, x, np.zeros(100)])
    # larger ragged case with empty rows and a dense row (edge cases)
    rng = np.random.default_rng(2025)
    rowptr, colind, values, _ = refc.random_csr(rng, 400, 300, 0.02)
    counts = np.diff(rowptr)
    counts[::7] = 0                       # force empty rows
    counts[5] = 300                       # one full (long) row
    rowptr = np.zeros(401, dtype=np.int64)
    rowptr[1:] = np.cumsum(counts)
    colind = np.concatenate([np.sort(rng.choice(300, size=int(c), replace=False)) for c in counts]
                            ).astype(np.int64)
    values = rng.uniform(-1.0, 1.0, rowptr[-1])
    save("spmv_ragged400", spmv, "spmv", [rowptr, colind, values, rng.uniform(-1, 1, 300),
                                          np.zeros(400)])
    # test_acceptance.py:99-117 — i64 values, exact
    sp = refc.spmv4_inputs()
    save("spmv_i64", parse(spmv_text(vt="i64")), "spmv",
         [sp[0], sp[1], np.array([1, 2, 3, 4, 5], dtype=np.int64),
          np.array([2, -3, 5, 7], dtype=np.int64), np.zeros(4, dtype=np.int64)])
    # i64 wraparound: products overflow 64 bits (interp.py:145-152)
    big = np.array([2**62 + 3, -(2**61) - 7, 2**40 + 1, 9, 2**63 - 1], dtype=np.int64)
    save("spmv_i64_wrap", parse(spmv_text(vt="i64")), "spmv",
         [sp[0], sp[1], big, np.array([5, 2**30 + 1, -3, 2**33], dtype=np.int64),
          np.zeros(4, dtype=np.int64)])
    # test_spmv_lowering.py:56-72 — i32 rowptr / colind get index casts
    save("spmv_i32idx", parse(spmv_text(rp="i32", ci="i32")), "spmv",
         [sp[0].astype(np.int32), sp[1].astype(np.int32), sp[2], sp[3], sp[4]])
    # f32 values (per-op float32 rounding, interp.py:155-160)
    rng = np.random.default_rng(7)
    rowptr, colind, values, _ = refc.random_csr(rng, 200, 150, 0.1)
    save("spmv_f32", parse(spmv_text(ci="i32", vt="f32")), "spmv",
         [rowptr, colind.astype(np.int32), values.astype(np.float32),
          rng.uniform(-1, 1, 150).astype(np.float32), np.zeros(200, dtype=np.float32)])
    # test_loop_mapping.py:150-162 / test_acceptance.py:194-205 — hint 16 at mean 14.34
    rng = np.random.default_rng(1465)
    rowptr, colind, values = refc.csr_with_mean(rng, 300, int(round(14.34 * 300)), 2048)
    save("spmv_mean1434", spmv, "spmv",
         [rowptr, colind, values, rng.uniform(-1, 1, 2048), np.zeros(300)])
    # empty matrix: zero rows (hint guard maxsi(N, 1), loop_mapping.py:238-240)
    save("spmv_empty", spmv, "spmv",
         [np.zeros(1, dtype=np.int64), np.zeros(0, dtype=np.int64), np.zeros(0), np.zeros(3),
          np.zeros(0)])
    # all rows empty
    save("spmv_allempty", spmv, "spmv",
         [np.zeros(6, dtype=np.int64), np.zeros(0, dtype=np.int64), np.zeros(0), np.ones(5),
          np.zeros(5)])

    # --- dense: test_acceptance.py:121-146 ----------------------------------------------
    rng = np.random.default_rng(5)
    a = rng.integers(-1000, 1000, (16, 16), dtype=np.int32)
    b = rng.integers(-1000, 1000, (16, 16), dtype=np.int32)
    save("matmul_i32", parse_file(str(REF / "tests/fixtures/matmul_i32.mlir")), "matmul", [a, b])
    af, bf = rng.uniform(-1, 1, (32, 32)), rng.uniform(-1, 1, (32, 32))
    mm64 = parse_file(str(REF / "tests/fixtures/matmul_f64.mlir"))
    save("matmul_f64", mm64, "matmul", [af, bf])
    # kernel-library route (linalg_lowering.py:32-45 -> kokkos.gemm), bit-exact to the loop route
    save("matmul_f64_kl", mm64, "matmul", [af, bf], kernel_library_calls=True)
    # dynamic-shape f32 / f64 (oracle/ir/matmul_*.mlir), ragged sizes, U(0,1) for f32
    rng = np.random.default_rng(3)
    for vt, dt in (("f32", np.float32), ("f64", np.float64)):
        m, n, k = 45, 70, 130
        A = rng.uniform(0, 1, (m, k)).astype(dt)
        B = rng.uniform(0, 1, (k, n)).astype(dt)
        save(f"matmul_dyn_{vt}", parse_file(str(IR / f"matmul_{vt}.mlir")), "matmul",
             [A, B, np.zeros((m, n), dtype=dt)])
    rng = np.random.default_rng(11)
    mv = parse_file(str(REF / "tests/fixtures/matvec_f64.mlir"))
    A, x = rng.uniform(-1, 1, (64, 64)), rng.uniform(-1, 1, 64)
    save("matvec_f64", mv, "matvec", [A, x])
    save("matvec_f64_kl", mv, "matvec", [A, x], kernel_library_calls=True)
    A, x = rng.uniform(-1, 1, (37, 300)), rng.uniform(-1, 1, 300)
    save("matvec_dyn", parse_file(str(IR / "matvec_f64.mlir")), "matvec", [A, x, np.zeros(37)])
    bmm = parse_file(str(REF / "tests/fixtures/batch_matmul_f32.mlir"))
    save("batch_matmul_f32", bmm, "bmm", refc.random_inputs(bmm, np.random.default_rng(12)))

    # --- parallel_reduce family (interp.py:174-195, 779-795) ----------------------------
    ar = parse_file(str(REF / "tests/fixtures/axis_reduce.mlir"))
    save("reduce_add_f64", ar, "rowsum", refc.random_inputs(ar, np.random.default_rng(13)))
    rng = np.random.default_rng(14)
    for comb in ("add", "mul", "min", "max"):
        for axes in ([1], [0]):
            src = rng.uniform(0.5, 1.5, (24, 40))
            save(f"reduce_{comb}_ax{axes[0]}_f64",
                 parse(reduce_text((24, 40), "f64", axes, comb)), "red", [src])
            srci = rng.integers(-9, 10, (24, 40)).astype(np.int64)
            save(f"reduce_{comb}_ax{axes[0]}_i64",
                 parse(reduce_text((24, 40), "i64", axes, comb)), "red", [srci])

    # --- SpMM / GCN loop nests (oracle/ir/*.mlir; no reference op) ------------
    rng = np.random.default_rng(21)
    rowptr, colind, values, _ = refc.random_csr(rng, 60, 50, 0.08)
    X = rng.uniform(-1, 1, (50, 8))
    save("spmm_k8", parse_file(str(IR / "spmm.mlir")), "spmm",
         [rowptr, colind.astype(np.int32), values, X, np.zeros((60, 8))])
    rng = np.random.default_rng(4)
    rowptr, colind, values, _ = refc.random_csr(rng, 40, 40, 0.1)
    values = np.abs(values).astype(np.float32)
    X = rng.uniform(0, 1, (40, 16)).astype(np.float32)
    W = rng.uniform(-1 / 8, 1 / 8, (16, 16)).astype(np.float32)
    save("gcn_small", parse_file(str(IR / "gcn_f32.mlir")), "gcn",
         [rowptr, colind.astype(np.int32), values, X, W, np.zeros((40, 16), dtype=np.float32)])


if __name__ == "__main__":
    main()
