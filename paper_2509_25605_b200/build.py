"""In-tree build of the CUDA backend: ``paper_2509_25605_b200/lib/liblapis_b200.so``.

Plain nvcc, sm_100a only (``-gencode arch=compute_100a,code=sm_100a``),
``-lineinfo`` for ncu source attribution.  The .so is git-ignored but travels
to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "lib"
SO = LIBDIR / "liblapis_b200.so"
INCLUDE = PKG.parent / "include"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills"]


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _compile(src: Path) -> Path:
    obj = LIBDIR / (src.stem + ".o")
    deps = [src, *CSRC.glob("*.cuh"), *INCLUDE.glob("*.h")]
    if _stale(obj, deps):
        cmd = [NVCC, *ARCH, *FLAGS, f"-I{INCLUDE}", "-c", str(src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src.name}:\n{r.stderr}")
        if r.stderr.strip():
            sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False) -> Path:
    LIBDIR.mkdir(exist_ok=True)
    srcs = sources()
    if force:
        for o in LIBDIR.glob("*.o"):
            o.unlink()
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(_compile, srcs))
    if force or _stale(SO, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", str(SO), *map(str, objs), "-lcudart", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
