"""Generate tests/golden/behavior/ — error, stale-access, configuration and
scalar-semantics cases for ``runtime.run`` — from the REFERENCE ITSELF.

    python tests/golden/make_behavior_golden.py

Each case is a small program written for this suite (the scenarios follow the
reference's own tests: test_interp.py stale reads / relaxed checking / sync
no-ops, test_acceptance.py error paths), optionally lowered by the reference
pipeline, run by ``lapis.interp.run`` under the given ExecConfig.  The npz
records the inputs and either the outputs + trace + counters or the raised
exception (class name and message).
"""
from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("LAPIS_REFERENCE", "/root/reference")) / "pkg"
sys.path.insert(0, str(REF / "src"))

from lapis.interp import ExecConfig, format_trace, run  # noqa: E402
from lapis.parser import parse  # noqa: E402
from lapis.passes import PassPipeline, TargetConfig, run_pipeline  # noqa: E402
from lapis.printer import print_program  # noqa: E402

OUT = Path(__file__).resolve().parent / "behavior"

STALE = """
func @f(%x: memref<4xf64, dualview>) -> (memref<4xf64, dualview>) {
  %c0 = arith.constant 0 : index
  %c1 = arith.constant 1 : index
  %n = arith.constant 4 : index
  %two = arith.constant 2.0 : f64
  kokkos.sync(%x) {space = device}
  kokkos.range_parallel (%i) in (%n) {executionSpace = device, parallelLevel = toprange} {
    %v = memref.load %x[%i]
    %w = arith.mulf(%v, %two)
    memref.store %w, %x[%i]
    kokkos.yield
  }
  kokkos.modify(%x) {space = device}
  %r = memref.load %x[%c0]
  memref.store %r, %x[%c1]
  func.return(%x)
}
"""

STALE_DEVICE = """
func @f(%x: memref<4xf64, dualview>, %y: memref<4xf64, dualview>) -> (memref<4xf64, dualview>) {
  %c0 = arith.constant 0 : index
  %n = arith.constant 4 : index
  %v9 = arith.constant 9.0 : f64
  kokkos.sync(%x) {space = device}
  memref.store %v9, %x[%c0]
  kokkos.modify(%x) {space = host}
  kokkos.range_parallel (%i) in (%n) {executionSpace = device, parallelLevel = toprange} {
    %v = memref.load %x[%i]
    memref.store %v, %y[%i]
    kokkos.yield
  }
  kokkos.modify(%y) {space = device}
  func.return(%y)
}
"""

DIV = """
func @f(%a: memref<?xi64>, %b: memref<?xi64>, %o: memref<?xi64>) -> (memref<?xi64>) {
  %c0 = arith.constant 0 : index
  %c1 = arith.constant 1 : index
  %n = memref.dim(%a) {index = 0}
  scf.parallel %i = %c0 to %n step %c1 {
    %x = memref.load %a[%i]
    %y = memref.load %b[%i]
    %q = arith.divi(%x, %y)
    %r = arith.ceildivsi(%x, %y)
    %s = arith.addi(%q, %r)
    memref.store %s, %o[%i]
    scf.yield
  }
  func.return(%o)
}
"""

INTSEM = """
func @f(%a: memref<?xi64>, %b: memref<?xi64>, %o: memref<?xi32>, %p: memref<?xi64>) -> (memref<?xi32>, memref<?xi64>) {
  %c0 = arith.constant 0 : index
  %c1 = arith.constant 1 : index
  %n = memref.dim(%a) {index = 0}
  %sh = arith.constant 3 : i64
  scf.parallel %i = %c0 to %n step %c1 {
    %x = memref.load %a[%i]
    %y = memref.load %b[%i]
    %m = arith.muli(%x, %y)
    %mi = arith.index_cast(%m) : index
    %t = arith.index_cast(%mi) : i32
    memref.store %t, %o[%i]
    %u = arith.cmpi(%x, %y) {predicate = ult}
    %sl = arith.shli(%x, %sh)
    %z = arith.select(%u, %sl, %m)
    %mx = arith.maxsi(%z, %y)
    memref.store %mx, %p[%i]
    scf.yield
  }
  func.return(%o, %p)
}
"""

DOT = """
func @dot(%x: memref<?xf64>, %y: memref<?xf64>) -> (f64) {
  %c0 = arith.constant 0 : index
  %c1 = arith.constant 1 : index
  %n = memref.dim(%x) {index = 0}
  %zero = arith.constant 0.0 : f64
  %s = scf.parallel %i = %c0 to %n step %c1 init(%zero) {
    %a = memref.load %x[%i]
    %b = memref.load %y[%i]
    %p = arith.mulf(%a, %b)
    scf.reduce(%p) {
      ^(%u: f64, %v: f64):
        %w = arith.addf(%u, %v)
        scf.reduce.return(%w)
    }
  }
  func.return(%s)
}
"""

MAXABS2D = """
func @m(%x: memref<?x?xf64>) -> (f64) {
  %c0 = arith.constant 0 : index
  %c1 = arith.constant 1 : index
  %r = memref.dim(%x) {index = 0}
  %c = memref.dim(%x) {index = 1}
  %lo = arith.constant -1.0e300 : f64
  %s = scf.parallel (%i, %j) = (%c0, %c0) to (%r, %c) step (%c1, %c1) init(%lo) {
    %a = memref.load %x[%i, %j]
    scf.reduce(%a) {
      ^(%u: f64, %v: f64):
        %g = arith.cmpf(%u, %v) {predicate = ogt}
        %w = arith.select(%g, %u, %v)
        scf.reduce.return(%w)
    }
  }
  func.return(%s)
}
"""

CUSTOM = """
func @c(%x: memref<?xf64>) -> (f64) {
  %c0 = arith.constant 0 : index
  %c1 = arith.constant 1 : index
  %n = memref.dim(%x) {index = 0}
  %one = arith.constant 1.0 : f64
  %s = scf.parallel %i = %c0 to %n step %c1 init(%one) {
    %a = memref.load %x[%i]
    scf.reduce(%a) {
      ^(%u: f64, %v: f64):
        %w = arith.subf(%u, %v)
        scf.reduce.return(%w)
    }
  }
  func.return(%s)
}
"""

DEVICE_SPACE = """
func @f(%x: memref<4xf64, dualview>) -> (f64) {
  %c0 = arith.constant 0 : index
  %n = arith.constant 4 : index
  %t = memref.alloc() : memref<4xf64, device>
  kokkos.sync(%x) {space = device}
  kokkos.range_parallel (%i) in (%n) {executionSpace = device, parallelLevel = toprange} {
    %v = memref.load %x[%i]
    memref.store %v, %t[%i]
    kokkos.yield
  }
  %r = memref.load %t[%c0]
  func.return(%r)
}
"""

SUBVIEW = """
func @f(%x: memref<8xf64>) -> (f64, memref<8xf64>) {
  %c2 = arith.constant 2 : index
  %c4 = arith.constant 4 : index
  %c1 = arith.constant 1 : index
  %c3 = arith.constant 3 : index
  %c0 = arith.constant 0 : index
  %v = arith.constant 42.0 : f64
  %sub = memref.subview %x[%c2][%c4]
  memref.store %v, %sub[%c1]
  scf.parallel %i = %c0 to %c4 step %c1 {
    %a = memref.load %sub[%i]
    %b = arith.addf(%a, %v)
    memref.store %b, %sub[%i]
    scf.yield
  }
  %out = memref.load %x[%c3]
  func.return(%out, %x)
}
"""


def spmv_program():
    return parse("""
    func @spmv(%rowptr: memref<?xindex>, %colind: memref<?xindex>, %values: memref<?xf64>,
               %x: memref<?xf64>, %y: memref<?xf64>) -> (memref<?xf64>) {
      sparse.spmv_csr(%rowptr, %colind, %values, %x, %y)
      func.return(%y)
    }""")


def lower(p):
    return run_pipeline(p, PassPipeline.preset(), TargetConfig()).program


def cases():
    rng = np.random.default_rng(5)
    spmv_bad_col = [np.array([0, 2, 3, 3, 5]), np.array([0, 1, 9, 0, 3]),
                    np.arange(1.0, 6.0), np.ones(4), np.zeros(4)]
    spmv_bad_range = [np.array([0, 2, 3, 3, 7]), np.array([0, 1, 2, 0, 3]),
                      np.arange(1.0, 6.0), np.ones(4), np.zeros(4)]
    spmv_decreasing = [np.array([0, 2, 1, 3, 5]), np.array([0, 1, 2, 0, 3]),
                       np.arange(1.0, 6.0), np.ones(4), np.zeros(4)]
    big = np.array([-(1 << 63), 7, -7, 5, 1 << 40, -3])
    yield "stale_host_strict", parse(STALE), "f", [np.ones(4)], ExecConfig()
    yield "stale_host_relaxed", parse(STALE), "f", [np.ones(4)], ExecConfig(strict_stale_checking=False)
    yield "stale_device_strict", parse(STALE_DEVICE), "f", [np.ones(4), np.zeros(4)], ExecConfig()
    yield "stale_device_relaxed", parse(STALE_DEVICE), "f", [np.ones(4), np.zeros(4)], \
        ExecConfig(strict_stale_checking=False)
    yield "single_memory", lower(spmv_program()), "spmv", \
        [np.array([0, 2, 3, 3, 5]), np.array([0, 1, 2, 0, 3]), np.arange(1.0, 6.0), np.ones(4),
         np.zeros(4)], ExecConfig(has_separate_device_memory=False)
    yield "spmv_bad_column", lower(spmv_program()), "spmv", spmv_bad_col, ExecConfig()
    yield "spmv_bad_column_orig", spmv_program(), "spmv", spmv_bad_col, ExecConfig()
    yield "spmv_bad_range", lower(spmv_program()), "spmv", spmv_bad_range, ExecConfig()
    yield "spmv_decreasing_rowptr", lower(spmv_program()), "spmv", spmv_decreasing, ExecConfig()
    yield "spmv_decreasing_orig", spmv_program(), "spmv", spmv_decreasing, ExecConfig()
    yield "div_ok", lower(parse(DIV)), "f", [big, np.array([-1, 2, 2, -2, 3, 7]), np.zeros(6, np.int64)], \
        ExecConfig()
    yield "div_by_zero", lower(parse(DIV)), "f", [big, np.array([-1, 2, 0, -2, 3, 7]),
                                                  np.zeros(6, np.int64)], ExecConfig()
    yield "int_semantics", lower(parse(INTSEM)), "f", \
        [np.array([1 << 62, -5, 3, 1 << 33, -(1 << 63), 9]), np.array([4, 3, -2, 1 << 31, -1, 9]),
         np.zeros(6, np.int32), np.zeros(6, np.int64)], ExecConfig()
    yield "dot_top_reduce", lower(parse(DOT)), "dot", [rng.uniform(-1, 1, 1000), rng.uniform(-1, 1, 1000)], \
        ExecConfig()
    yield "dot_orig", parse(DOT), "dot", [rng.uniform(-1, 1, 300), rng.uniform(-1, 1, 300)], ExecConfig()
    yield "max_2d_reduce", lower(parse(MAXABS2D)), "m", [rng.uniform(-5, 5, (37, 13))], ExecConfig()
    yield "custom_combiner", lower(parse(CUSTOM)), "c", [rng.uniform(0, 1, 50)], ExecConfig()
    yield "device_space_host_read", parse(DEVICE_SPACE), "f", [np.ones(4)], ExecConfig()
    yield "subview_alias", lower(parse(SUBVIEW)), "f", [np.arange(8.0)], ExecConfig()
    yield "empty_rows", lower(spmv_program()), "spmv", \
        [np.zeros(6, np.int64), np.zeros(0, np.int64), np.zeros(0), np.ones(3), np.full(5, 7.0)], \
        ExecConfig()


def main() -> None:
    OUT.mkdir(exist_ok=True)
    for name, program, entry, inputs, config in cases():
        arrays = {f"in{i}": np.asarray(a) for i, a in enumerate(inputs)}
        arrays["entry"] = np.array(entry)
        arrays["config"] = np.array(json.dumps({
            "strict_stale_checking": config.strict_stale_checking,
            "has_separate_device_memory": config.has_separate_device_memory}))
        try:
            r = run(program, entry, [np.array(a, copy=True) for a in inputs], config)
            for i, o in enumerate(r.outputs):
                arrays[f"out{i}"] = np.asarray(o)
            arrays["trace"] = np.array(format_trace(r.trace))
            arrays["counters"] = np.array(json.dumps({k: dict(v) for k, v in r.counters.items()},
                                                     sort_keys=True))
            arrays["error"] = np.array("")
        except Exception as e:  # the reference's own error behaviour is the golden
            arrays["error"] = np.array(f"{type(e).__name__}: {e}")
        (OUT / f"{name}.mlir").write_text(print_program(program))
        np.savez(OUT / f"{name}.npz", **arrays)
        print(name, str(arrays["error"]) or "ok")


if __name__ == "__main__":
    main()
