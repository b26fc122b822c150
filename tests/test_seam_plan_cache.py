"""LAPIS::spmv_csr's structure-plan cache (include/lapis_b200_runtime.hpp
b200::CsrPlanCache): the emitted C++ seam (golden cpp/spmv.hpp:16-70 calls
LAPIS::spmv_csr) builds a reference-order plan on the first call whose rowptr
DualView has no pending modification, replays it afterwards, and drops it when
rowptr is modified.  Every call is bit-identical to the oracle's sequential
row sums (interp.py:808-811)."""
from pathlib import Path

import numpy as np
import pytest

import cxx_drivers as D
from matrices import stencil_csr
from oracle import oracle as O

DRIVER = r"""
#include "lapis_b200_runtime.hpp"
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>
template <class T> static std::vector<T> slurp(const std::string& p, size_t n) {
  std::vector<T> v(n); std::ifstream f(p, std::ios::binary);
  if (!f.read(reinterpret_cast<char*>(v.data()), n * sizeof(T))) std::exit(3);
  return v; }
template <class T> static void dump(const std::string& p, LAPIS::DualView<T*>& y) {
  y.syncHost(); auto h = y.host_view(); std::ofstream o(p, std::ios::binary);
  for (int64_t i = 0; i < (int64_t)h.extent(0); ++i) o.write((const char*)&h(i), sizeof(T)); }
int main(int argc, char** argv) {
  const std::string dir = argv[1];
  const int64_t n = std::atoll(argv[2]), nnz = std::atoll(argv[3]);
  Kokkos::initialize();
  {
    auto rp = slurp<int64_t>(dir + "/rp.bin", n + 1);
    auto ci = slurp<int32_t>(dir + "/ci.bin", nnz);
    auto va = slurp<double>(dir + "/va.bin", nnz);
    auto xx = slurp<double>(dir + "/x.bin", n);
    auto rp2 = slurp<int64_t>(dir + "/rp2.bin", n + 1);
    LAPIS::DualView<int64_t*> R("rp", n + 1);
    LAPIS::DualView<int32_t*> C("ci", nnz);
    LAPIS::DualView<double*> V("va", nnz), X("x", n), Y("y", n);
    for (int64_t i = 0; i <= n; ++i) R.host_view()(i) = rp[i];
    for (int64_t i = 0; i < nnz; ++i) { C.host_view()(i) = ci[i]; V.host_view()(i) = va[i]; }
    for (int64_t i = 0; i < n; ++i) X.host_view()(i) = xx[i];
    R.modifyHost(); C.modifyHost(); V.modifyHost(); X.modifyHost();
    using LAPIS::b200::csr_plan_cache_size;
    LAPIS::spmv_csr(R, C, V, X, Y);  // rowptr host-modified: the no-plan call
    std::printf("cache1=%zu\n", csr_plan_cache_size()); dump(dir + "/y1.bin", Y);
    LAPIS::spmv_csr(R, C, V, X, Y);  // builds the plan
    std::printf("cache2=%zu\n", csr_plan_cache_size()); dump(dir + "/y2.bin", Y);
    LAPIS::spmv_csr(R, C, V, X, Y);  // replays it
    std::printf("cache3=%zu\n", csr_plan_cache_size()); dump(dir + "/y3.bin", Y);
    for (int64_t i = 0; i <= n; ++i) R.host_view()(i) = rp2[i];  // a new structure
    R.modifyHost();
    LAPIS::spmv_csr(R, C, V, X, Y);  // drops the stale plan
    std::printf("cache4=%zu\n", csr_plan_cache_size()); dump(dir + "/y4.bin", Y);
    LAPIS::spmv_csr(R, C, V, X, Y);  // plan of the new structure
    std::printf("cache5=%zu\n", csr_plan_cache_size()); dump(dir + "/y5.bin", Y);
  }
  Kokkos::finalize();
  return 0;
}
"""


def _build(tmp_path, compile_only):
    src = tmp_path / "seam_cache.cu"
    src.write_text(DRIVER)
    exe = tmp_path / ("seam_cache.o" if compile_only else "seam_cache")
    r = D.compile_driver(src, exe, compile_only=compile_only, b200_seam=True)
    assert r.returncode == 0, r.stderr[-3000:]
    return exe


@pytest.mark.skipif(D.nvcc() is None or not D.emitted_cases(), reason="no nvcc / runtime header")
def test_seam_cache_compiles(tmp_path):
    _build(tmp_path, compile_only=True)


@pytest.mark.gpu
@pytest.mark.skipif(D.nvcc() is None or not D.emitted_cases(), reason="no nvcc / runtime header")
def test_seam_cache_replays_and_invalidates(tmp_path, cuda_device):
    import subprocess
    exe = _build(tmp_path, compile_only=False)
    rp, ci, va = stencil_csr(27, 40)      # 64000 rows: the row-stream plan
    n, nnz = rp.size - 1, int(rp[-1])
    x = np.random.default_rng(4).uniform(-1, 1, n)
    # second structure: the same arrays with every row past n/2 empty
    rp2 = np.minimum(rp, rp[n // 2])
    for name, a in (("rp", rp), ("ci", ci.astype(np.int32)), ("va", va), ("x", x), ("rp2", rp2)):
        np.ascontiguousarray(a).tofile(tmp_path / f"{name}.bin")
    r = subprocess.run([str(exe), str(tmp_path), str(n), str(nnz)], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    sizes = dict(line.split("=") for line in r.stdout.split() if line.startswith("cache"))
    assert sizes == {"cache1": "0", "cache2": "1", "cache3": "1", "cache4": "0", "cache5": "1"}, r.stdout
    y = {i: np.fromfile(tmp_path / f"y{i}.bin", dtype=np.float64) for i in range(1, 6)}
    want = O.spmv_csr(rp, ci, va, x)
    want2 = O.spmv_csr(rp2, ci, va, x)
    for i in (1, 2, 3):
        assert np.array_equal(y[i].view(np.uint64), want.view(np.uint64)), i
    for i in (4, 5):
        assert np.array_equal(y[i].view(np.uint64), want2.view(np.uint64)), i
