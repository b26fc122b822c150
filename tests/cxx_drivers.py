"""Drivers for the reference-emitted Kokkos C++ compiled against the B200
Kokkos subset (include/kokkos_b200/Kokkos_Core.hpp) — TEST INFRASTRUCTURE.

For one drop-in case (tests/golden/run/<name>) the driver
  * reads every argument from a raw little-endian file (the reference's
    `file:` args convention, tensors.py:25-104), builds a host View and adopts
    it into a LAPIS::DualView (host-modified, as interp.run's inputs are);
  * calls the emitted function exactly as the emitted signature declares it;
  * syncs the result to the host and writes it raw, then prints the
    LAPIS::transferStats() counters.
"""
from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
EMITTED = ROOT / "oracle" / "_ref" / "emitted"
KOKKOS_B200 = ROOT / "include" / "kokkos_b200"
CTYPE = {"f32": "float", "f64": "double", "i32": "int32_t", "i64": "int64_t", "index": "int64_t",
         "i1": "bool"}


def emitted_cases() -> list[str]:
    idx = EMITTED / "index.txt"
    return idx.read_text().split() if idx.exists() else []


def nvcc() -> str | None:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and Path(c).exists():
            return c
    return None


def driver_source(name: str, program, entry: str, inputs: list, b200_seam: bool = False) -> str:
    """C++ driver for `entry` of the (lowered) program with these inputs.
    ``b200_seam``: include include/lapis_b200_runtime.hpp first, so the emitted
    LAPIS::gemm / gemv calls resolve to the B200 kernels."""
    from lapis.ir import MemRefType, func_result_types
    func = program.find_func(entry)
    params = func.region(0).args
    lines = (['#include "lapis_b200_runtime.hpp"'] if b200_seam else []) + [
             f'#include "{name}.hpp"', "#include <algorithm>", "#include <cstdio>",
             "#include <fstream>", "#include <string>", "#include <vector>",
             "template <class T> static std::vector<T> slurp(const std::string& p, size_t n) {",
             "  std::vector<T> v(n ? n : 1); std::ifstream f(p, std::ios::binary);",
             "  if (n && !f.read(reinterpret_cast<char*>(v.data()), n * sizeof(T))) {"
             " std::fprintf(stderr, \"read %s\\n\", p.c_str()); std::exit(3); }",
             "  return v; }",
             "int main(int argc, char** argv) {",
             "  const std::string dir = argc > 1 ? argv[1] : \".\";",
             "  lapis_initialize();", "  {"]
    args = []
    for i, (p, a) in enumerate(zip(params, inputs)):
        t = p.type
        if isinstance(t, MemRefType):
            ct = CTYPE[t.element.kind]
            shape = list(np.asarray(a).shape)
            n = int(np.prod(shape)) if shape else 1
            stars = "*" * len(shape)
            ext = ", ".join(str(d) for d in shape)
            lines.append(f'    auto d{i} = slurp<{ct}>(dir + "/in{i}.bin", {n});')
            lines.append(f'    Kokkos::View<{ct}{stars}, Kokkos::LayoutRight, Kokkos::HostSpace> '
                         f'h{i}("arg{i}"' + (f", {ext}" if ext else "") + ");")
            lines.append(f"    std::copy(d{i}.begin(), d{i}.begin() + {n}, h{i}.data());")
            lines.append(f"    LAPIS::DualView<{ct}{stars}> a{i}(h{i});")
            args.append(f"a{i}")
        else:
            v = np.asarray(a).item()
            args.append(repr(float(v)) if t.kind in ("f32", "f64") else f"INT64_C({int(v)})")
    res = func_result_types(func)
    lines.append(f"    auto r = {entry}({', '.join(args)});")
    lines.append('    std::ofstream o(dir + "/out0.bin", std::ios::binary);')
    if res and isinstance(res[0], MemRefType):
        t = res[0]
        ct = CTYPE[t.element.kind]
        lines.append("    r.syncHost();")
        lines.append("    auto hv = r.host_view();")
        ivs = [f"i{d}" for d in range(t.rank)]
        for d, iv in enumerate(ivs):
            lines.append("    " + "  " * d +
                         f"for (int64_t {iv} = 0; {iv} < (int64_t)hv.extent({d}); ++{iv}) {{")
        lines.append("    " + "  " * t.rank + f"{ct} v = hv({', '.join(ivs)}); "
                     "o.write(reinterpret_cast<const char*>(&v), sizeof(v));")
        for d in range(t.rank - 1, -1, -1):
            lines.append("    " + "  " * d + "}")
    elif res:
        ct = CTYPE[res[0].kind]
        lines.append(f"    {ct} v = r; o.write(reinterpret_cast<const char*>(&v), sizeof(v));")
    lines.append("  }")
    lines.append('  std::printf("h2d_count=%zu d2h_count=%zu h2d_bytes=%zu d2h_bytes=%zu\\n", '
                 "LAPIS::transferStats().h2d_count, LAPIS::transferStats().d2h_count, "
                 "LAPIS::transferStats().h2d_bytes, LAPIS::transferStats().d2h_bytes);")
    lines.append("  lapis_finalize();")
    lines.append("  return 0;")
    lines.append("}")
    return "\n".join(lines) + "\n"


LIBDIR = ROOT / "paper_2509_25605_b200" / "lib"


def compile_driver(src: Path, out: Path, compile_only: bool = False,
                   b200_seam: bool = False, extra_include: Path | None = None
                   ) -> subprocess.CompletedProcess:
    inc = [f"-I{extra_include}"] if extra_include else []
    cmd = [nvcc(), "-std=c++17", "-O2", "-gencode", "arch=compute_100a,code=sm_100a",
           "--extended-lambda", "-w", f"-I{KOKKOS_B200}", *inc, f"-I{EMITTED}",
           f"-I{ROOT / 'include'}", "-x", "cu"]
    cmd += (["-c", str(src), "-o", str(out)] if compile_only else [str(src), "-o", str(out)])
    if b200_seam and not compile_only:
        cmd += [f"-L{LIBDIR}", "-llapis_b200", f"-Xlinker=-rpath,{LIBDIR}"]
    return subprocess.run(cmd, capture_output=True, text=True)


NPTYPE = {"f32": np.float32, "f64": np.float64, "i32": np.int32, "i64": np.int64,
          "index": np.int64, "i1": np.bool_}


def coerce_inputs(program, entry: str, inputs: list) -> list:
    """Arrays in the element type of each memref parameter (what interp.run's
    coerce_scalar does element by element, interp.py:330-353)."""
    from lapis.ir import MemRefType
    out = []
    for p, a in zip(program.find_func(entry).region(0).args, inputs):
        out.append(np.asarray(a).astype(NPTYPE[p.type.element.kind])
                   if isinstance(p.type, MemRefType) else a)
    return out


def write_inputs(d: Path, inputs: list) -> None:
    for i, a in enumerate(inputs):
        np.ascontiguousarray(a).tofile(d / f"in{i}.bin")


def read_output(d: Path, like: np.ndarray) -> np.ndarray:
    return np.fromfile(d / "out0.bin", dtype=like.dtype).reshape(like.shape)
