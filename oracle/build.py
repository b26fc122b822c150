"""Build recipe for the checker side (TEST INFRASTRUCTURE ONLY).

1. ``oracle/liblapis_oracle.so`` — the C restatement ``oracle/lapis_oracle.c``
   (gcc, ``-ffp-contract=off`` so no multiply-add is fused, OpenMP over rows).
2. ``oracle/_ref/liblapis_ref.so`` — the reference's OWN CPU path for the hot
   kernels, built only when ``/root/reference`` is present (this container;
   the GPU box uses the prebuilt file, which travels with the snapshot):

   * the reference CLI (``python -m lapis.cli``, imported from
     ``/root/reference/pkg/src``) lowers each IR file with the preset
     ``--sparse-compiler-kokkos`` pipeline and emits Kokkos C++ into
     ``oracle/_ref/<name>.hpp`` plus the runtime header
     (``--emit-runtime-header``);
   * ``oracle/ref_driver.cpp`` is compiled once per emitted header with g++
     against the reference's serial Kokkos stub
     (``/root/reference/pkg/cxx_runtime/include``, ``-DLAPIS_USE_SERIAL_STUB``)
     and ``-ffp-contract=off`` (bit-identical to the interpreter);
   * the objects are linked into one shared library.

Nothing is copied out of /root/reference: sources are compiled where they lie
and every output goes to ``oracle/_ref/`` (git-ignored).
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF_ROOT = Path(os.environ.get("LAPIS_REFERENCE", "/root/reference"))
REF_PKG = REF_ROOT / "pkg"
OUT = HERE / "_ref"
ORACLE_SO = HERE / "liblapis_oracle.so"
# -march=native (SURVEY 8(d) CPU recipe) build, recorded with the ISA flags of
# the build host: oracle/ref.py loads it only on a host whose CPU has every one
# of them (the GPU box's CPU may differ from this one), else the portable
# build of the same objects
REF_SO_NATIVE = OUT / "liblapis_ref.so"
REF_SO = OUT / "liblapis_ref_portable.so"
NATIVE_FLAGS = OUT / "native_cpu_flags.txt"


def cpu_flags() -> set:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("flags"):
                return set(line.split(":", 1)[1].split())
    except OSError:
        pass
    return set()

# (header name, IR source, REF_KIND, value type, colind type, entry symbol)
#   REF_KIND: 1 spmv, 2 spmm, 3 matmul, 4 matvec, 5 gcn
REF_UNITS = [
    # the reference's own fixture: index (int64) rowptr and colind, f64
    ("spmv_ref", REF_PKG / "tests/fixtures/spmv.mlir", 1, "double", "int64_t", "ref_spmv_f64_i64"),
    ("spmv_i32", HERE / "ir/spmv_i32.mlir", 1, "double", "int32_t", "ref_spmv_f64_i32"),
    ("spmm", HERE / "ir/spmm.mlir", 2, "double", "int32_t", "ref_spmm_f64_i32"),
    ("gcn_f32", HERE / "ir/gcn_f32.mlir", 5, "float", "int32_t", "ref_gcn_f32_i32"),
    ("matmul_f32", HERE / "ir/matmul_f32.mlir", 3, "float", "int32_t", "ref_matmul_f32"),
    ("matmul_f64", HERE / "ir/matmul_f64.mlir", 3, "double", "int32_t", "ref_matmul_f64"),
    ("matvec_f64", HERE / "ir/matvec_f64.mlir", 4, "double", "int32_t", "ref_matvec_f64"),
]


def _run(cmd, **kw):
    r = subprocess.run(cmd, capture_output=True, text=True, **kw)
    if r.returncode != 0:
        raise RuntimeError(f"command failed ({r.returncode}): {' '.join(map(str, cmd))}\n"
                           f"{r.stdout}\n{r.stderr}")
    return r.stdout


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).exists() and Path(d).stat().st_mtime > t for d in deps)


def build_oracle(force: bool = False) -> Path:
    src = HERE / "lapis_oracle.c"
    if force or _stale(ORACLE_SO, [src, __file__]):
        _run(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
              "-std=c11", str(src), "-o", str(ORACLE_SO), "-lm"])
    return ORACLE_SO


def reference_available() -> bool:
    return (REF_PKG / "src/lapis/cli.py").exists() and \
        (REF_PKG / "cxx_runtime/include/lapis_serial_stub.hpp").exists()


def _lapis_cli(args, stdin_text=None):
    env = dict(os.environ)
    env["PYTHONPATH"] = str(REF_PKG / "src") + os.pathsep + env.get("PYTHONPATH", "")
    r = subprocess.run([sys.executable, "-m", "lapis.cli", *args], input=stdin_text,
                       capture_output=True, text=True, env=env)
    if r.returncode != 0:
        raise RuntimeError(f"lapis {' '.join(args)} failed: {r.stderr}")
    return r.stdout


def build_reference(force: bool = False) -> Path | None:
    if not reference_available():
        return REF_SO if REF_SO.exists() else None
    OUT.mkdir(exist_ok=True)
    driver = HERE / "ref_driver.cpp"
    deps = [driver, __file__, *(u[1] for u in REF_UNITS)]
    if not force and not _stale(REF_SO, deps) and not _stale(REF_SO_NATIVE, deps):
        return REF_SO_NATIVE
    runtime_hdr = OUT / "lapis_dualview_runtime.hpp"
    variants = {REF_SO: [], REF_SO_NATIVE: ["-march=native"]}   # portable, native
    objs = {so: [] for so in variants}
    for name, ir, kind, vt, ct, entry in REF_UNITS:
        lowered = _lapis_cli(["opt", "--sparse-compiler-kokkos", str(ir)])
        (OUT / f"{name}.mlir").write_text(lowered)
        _lapis_cli(["translate", "--header-name", name, "--emit-runtime-header", str(runtime_hdr),
                    "-o", str(OUT / f"{name}.hpp"), str(OUT / f"{name}.mlir")])
        for so, extra in variants.items():
            obj = OUT / f"{name}{'_native' if extra else ''}.o"
            cmd = ["g++", "-std=c++17", "-O3", *extra, "-ffp-contract=off", "-fPIC", "-pthread",
                   "-DLAPIS_USE_SERIAL_STUB", f"-I{OUT}", f"-I{REF_PKG / 'cxx_runtime/include'}",
                   f'-DREF_HEADER="{name}.hpp"', f"-DREF_KIND={kind}", f"-DREF_VT={vt}",
                   f"-DREF_CT={ct}", f"-DREF_ENTRY={entry}"]
            if name == "spmv_ref":
                cmd.append("-DREF_TRANSFER_PROBE")
            _run(cmd + ["-c", str(driver), "-o", str(obj)])
            objs[so].append(str(obj))
    for so in variants:
        _run(["g++", "-shared", "-pthread", "-o", str(so), *objs[so]])
    NATIVE_FLAGS.write_text(" ".join(sorted(cpu_flags())) + "\n")
    return REF_SO_NATIVE


EMITTED = OUT / "emitted"
RUN_GOLDEN = HERE.parent / "tests" / "golden" / "run"


def emit_run_cases(force: bool = False) -> list:
    """The reference emitter's Kokkos C++ for every lowered drop-in case
    (tests/golden/run/*.lowered.mlir) -> oracle/_ref/emitted/<name>.hpp, plus
    the runtime header.  Compiled on the GPU box against
    include/kokkos_b200/Kokkos_Core.hpp by tests/test_kokkos_b200_gpu.py.
    Cases the reference emitter rejects are skipped (listed in index.txt)."""
    if not reference_available():
        return []
    EMITTED.mkdir(parents=True, exist_ok=True)
    index = EMITTED / "index.txt"
    srcs = sorted(RUN_GOLDEN.glob("*.lowered.mlir"))
    if not force and index.exists() and not _stale(index, [*srcs, __file__]):
        return index.read_text().split()
    ok = []
    for src in srcs:
        name = src.name[: -len(".lowered.mlir")]
        try:
            _lapis_cli(["translate", "--header-name", name, "--emit-runtime-header",
                        str(EMITTED / "lapis_dualview_runtime.hpp"), "-o",
                        str(EMITTED / f"{name}.hpp"), str(src)])
            ok.append(name)
        except RuntimeError:
            continue
    index.write_text("\n".join(ok) + "\n")
    return ok


def main() -> None:
    force = "--force" in sys.argv
    print("oracle:", build_oracle(force))
    ref = build_reference(force)
    print("reference CPU path:", ref if ref else "unavailable (no /root/reference and no prebuilt)")
    print("emitted C++ cases:", len(emit_run_cases(force)))


if __name__ == "__main__":
    main()
