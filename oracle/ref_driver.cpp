// ref_driver.cpp — drives the reference's OWN emitted Kokkos C++ on the
// reference's OWN serial Kokkos stub, behind extern "C" entry points that
// oracle/ref.py loads with ctypes.
//
// TEST / BASELINE INFRASTRUCTURE ONLY (oracle/ is never imported by the
// product package).  The kernel bodies are not in this file: each
// translation unit #includes one header that the reference CLI emitted into
// oracle/_ref/ (`lapis opt --sparse-compiler-kokkos | lapis translate`), and
// that header #includes the reference runtime header (DualView, emitted by
// `lapis translate --emit-runtime-header`) and the reference serial stub
// /root/reference/pkg/cxx_runtime/include/lapis_serial_stub.hpp
// (-DLAPIS_USE_SERIAL_STUB).  See oracle/build.py for the recipe.
//
// Structure of each entry (modelled on the reference's
// pkg/cxx_runtime/drivers/spmv_driver.cpp:9-54): fill host views, mark them
// host-modified, call the emitted function once (the lazy syncDevice copies
// happen here, runtime_header.py:152-164), then time `reps` further calls
// (no copies: the host side is clean) and read the result back with syncHost.
//
// `threads` > 1 splits the OUTER row range into contiguous blocks, one
// std::thread each, every block running the unmodified emitted function on
// its own DualViews (rowptr rebased, colind global, x / B replicated), i.e.
// data decomposition around the serial reference code.  Per-row summation
// order is untouched, so the output is bitwise identical to threads == 1
// (checked by tests/test_ref_path.py).
#include REF_HEADER

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace {

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

template <class F>
void run_blocks(int nblk, F f) {
  if (nblk <= 1) { f(0); return; }
  std::vector<std::thread> ts;
  ts.reserve(nblk);
  for (int b = 0; b < nblk; ++b) ts.emplace_back([&, b] { f(b); });
  for (auto& t : ts) t.join();
}

template <class T>
void fill1(LAPIS::DualView<T*>& dv, const T* src, int64_t n) {
  auto h = dv.host_view();
  for (int64_t i = 0; i < n; ++i) h(i) = src[i];
  dv.modifyHost();
}

template <class T>
void fill2(LAPIS::DualView<T**>& dv, const T* src, int64_t rows, int64_t cols, int64_t ld) {
  auto h = dv.host_view();
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j) h(i, j) = src[i * ld + j];
  dv.modifyHost();
}

}  // namespace

#if REF_KIND == 1 || REF_KIND == 2 || REF_KIND == 5
// ---------------------------------------------------------------- CSR kernels
// REF_VT: value type; REF_CT: colind element type of the emitted signature.
// Everything driver-local lives in an anonymous namespace: several of these
// translation units are linked into one .so and their Block layouts differ.
namespace {
struct Block {
  int64_t r0, r1;
  LAPIS::DualView<int64_t*> rp;
  LAPIS::DualView<REF_CT*> ci;
  LAPIS::DualView<REF_VT*> v;
#if REF_KIND == 1
  LAPIS::DualView<REF_VT*> x, y;
#else
  LAPIS::DualView<REF_VT**> x, y;
#endif
#if REF_KIND == 5
  LAPIS::DualView<REF_VT**> w;
#endif
};

static std::vector<Block> make_blocks(int64_t nrows, int64_t ncols, int64_t k, int64_t kout,
                                      const int64_t* rowptr, const REF_CT* colind,
                                      const REF_VT* values, const REF_VT* x, const REF_VT* w,
                                      int nblk) {
  std::vector<Block> bl(nblk);
  for (int b = 0; b < nblk; ++b) {
    Block& B = bl[b];
    B.r0 = nrows * b / nblk;
    B.r1 = nrows * (b + 1) / nblk;
    const int64_t n = B.r1 - B.r0, base = rowptr[B.r0], nnz = rowptr[B.r1] - base;
    B.rp = LAPIS::DualView<int64_t*>("rowptr", n + 1);
    {
      auto h = B.rp.host_view();
      for (int64_t i = 0; i <= n; ++i) h(i) = rowptr[B.r0 + i] - base;
      B.rp.modifyHost();
    }
    B.ci = LAPIS::DualView<REF_CT*>("colind", nnz);
    B.v = LAPIS::DualView<REF_VT*>("values", nnz);
    fill1(B.v, values + base, nnz);
#if REF_KIND == 1
    (void)k; (void)kout;
    // x restricted to the block's column window [cmin, cmax], colind rebased by
    // cmin: the same products in the same order, without replicating all of x
    // per thread (the config-5 x is 1.6 GB).
    int64_t cmin = ncols, cmax = -1;
    for (int64_t j = 0; j < nnz; ++j) {
      const int64_t cj = (int64_t)colind[base + j];
      cmin = cj < cmin ? cj : cmin;
      cmax = cj > cmax ? cj : cmax;
    }
    if (cmax < cmin) { cmin = 0; cmax = -1; }
    {
      auto h = B.ci.host_view();
      for (int64_t j = 0; j < nnz; ++j) h(j) = (REF_CT)((int64_t)colind[base + j] - cmin);
      B.ci.modifyHost();
    }
    B.x = LAPIS::DualView<REF_VT*>("x", cmax - cmin + 1);
    fill1(B.x, x + cmin, cmax - cmin + 1);
    B.y = LAPIS::DualView<REF_VT*>("y", n);
    B.y.modifyHost();
#else
    // the block's referenced rows of X only, columns relabelled in ascending
    // order (a power-law block references columns all over X, so a window as
    // for SpMV would be the whole 5 GB operand per block): relabelling keeps
    // every row's entry sequence, hence the emitted sum, unchanged
    std::vector<int64_t> used(colind + base, colind + base + nnz);
    std::sort(used.begin(), used.end());
    used.erase(std::unique(used.begin(), used.end()), used.end());
    {
      auto h = B.ci.host_view();
      for (int64_t j = 0; j < nnz; ++j)
        h(j) = (REF_CT)(std::lower_bound(used.begin(), used.end(), (int64_t)colind[base + j]) -
                        used.begin());
      B.ci.modifyHost();
    }
    const int64_t nused = (int64_t)used.size();
    B.x = LAPIS::DualView<REF_VT**>("x", nused > 0 ? nused : 1, k);
    {
      auto h = B.x.host_view();
      for (int64_t i = 0; i < nused; ++i)
        for (int64_t j = 0; j < k; ++j) h(i, j) = x[used[i] * k + j];
      B.x.modifyHost();
    }
    (void)ncols;
#if REF_KIND == 5
    B.w = LAPIS::DualView<REF_VT**>("w", k, kout);
    fill2(B.w, w, k, kout, kout);
    B.y = LAPIS::DualView<REF_VT**>("h", n, kout);
#else
    (void)w; (void)kout;
    B.y = LAPIS::DualView<REF_VT**>("y", n, k);
#endif
    B.y.modifyHost();
#endif
  }
  return bl;
}

static void call_block(Block& B) {
#if REF_KIND == 1
  B.y = spmv(B.rp, B.ci, B.v, B.x, B.y);
#elif REF_KIND == 2
  B.y = spmm(B.rp, B.ci, B.v, B.x, B.y);
#else
  B.y = gcn(B.rp, B.ci, B.v, B.x, B.w, B.y);
#endif
}
}  // namespace

// Writes the wall time of each of `reps` timed calls (seconds) to times[] and
// the result rows to y (row-major).
extern "C" int REF_ENTRY(int64_t nrows, int64_t ncols, int64_t k, int64_t kout,
                         const int64_t* rowptr, const REF_CT* colind, const REF_VT* values,
                         const REF_VT* x, const REF_VT* w, REF_VT* y, int reps, int threads,
                         double* times) {
  lapis_initialize();
  int nblk = std::max(1, (int)std::min<int64_t>(threads, std::max<int64_t>(nrows, 1)));
  auto bl = make_blocks(nrows, ncols, k, kout, rowptr, colind, values, x, w, nblk);
  for (auto& B : bl) call_block(B);  // warm-up: lazy H2D copies happen here, serially
  for (int r = 0; r < reps; ++r) {
    double t0 = now_s();
    run_blocks(nblk, [&](int b) { call_block(bl[b]); });
    if (times) times[r] = now_s() - t0;
  }
  for (auto& B : bl) {
    B.y.syncHost();
    auto h = B.y.host_view();
    const int64_t n = B.r1 - B.r0;
#if REF_KIND == 1
    for (int64_t i = 0; i < n; ++i) y[B.r0 + i] = h(i);
#else
    const int64_t cols = (REF_KIND == 5) ? kout : k;
    for (int64_t i = 0; i < n; ++i)
      for (int64_t c = 0; c < cols; ++c) y[(B.r0 + i) * cols + c] = h(i, c);
#endif
  }
  lapis_finalize();
  return 0;
}

#elif REF_KIND == 3
// ------------------------------------------------------------ dense matmul
extern "C" int REF_ENTRY(int64_t m, int64_t n, int64_t k, const REF_VT* a, const REF_VT* b,
                         REF_VT* c, int reps, int threads, double* times) {
  lapis_initialize();
  int nblk = std::max(1, (int)std::min<int64_t>(threads, std::max<int64_t>(m, 1)));
  struct MB { int64_t r0, r1; LAPIS::DualView<REF_VT**> a, b, c; };
  std::vector<MB> bl(nblk);
  for (int t = 0; t < nblk; ++t) {
    MB& B = bl[t];
    B.r0 = m * t / nblk; B.r1 = m * (t + 1) / nblk;
    B.a = LAPIS::DualView<REF_VT**>("a", B.r1 - B.r0, k);
    fill2(B.a, a + B.r0 * k, B.r1 - B.r0, k, k);
    B.b = LAPIS::DualView<REF_VT**>("b", k, n);
    fill2(B.b, b, k, n, n);
    B.c = LAPIS::DualView<REF_VT**>("c", B.r1 - B.r0, n);
    B.c.modifyHost();
  }
  for (auto& B : bl) B.c = matmul(B.a, B.b, B.c);
  for (int r = 0; r < reps; ++r) {
    double t0 = now_s();
    run_blocks(nblk, [&](int t) { bl[t].c = matmul(bl[t].a, bl[t].b, bl[t].c); });
    if (times) times[r] = now_s() - t0;
  }
  for (auto& B : bl) {
    B.c.syncHost();
    auto h = B.c.host_view();
    for (int64_t i = 0; i < B.r1 - B.r0; ++i)
      for (int64_t j = 0; j < n; ++j) c[(B.r0 + i) * n + j] = h(i, j);
  }
  lapis_finalize();
  return 0;
}

#elif REF_KIND == 4
// ------------------------------------------------------------ dense matvec
extern "C" int REF_ENTRY(int64_t m, int64_t n, const REF_VT* a, const REF_VT* x, REF_VT* y,
                         int reps, double* times) {
  lapis_initialize();
  LAPIS::DualView<REF_VT**> A("a", m, n);
  fill2(A, a, m, n, n);
  LAPIS::DualView<REF_VT*> X("x", n);
  fill1(X, x, n);
  LAPIS::DualView<REF_VT*> Y("y", m);
  Y.modifyHost();
  Y = matvec(A, X, Y);
  for (int r = 0; r < reps; ++r) {
    double t0 = now_s();
    Y = matvec(A, X, Y);
    if (times) times[r] = now_s() - t0;
  }
  Y.syncHost();
  auto h = Y.host_view();
  for (int64_t i = 0; i < m; ++i) y[i] = h(i);
  lapis_finalize();
  return 0;
}
#endif

#if REF_KIND == 1 && defined(REF_TRANSFER_PROBE)
// Transfer-counter probe for the 4x4 fixture (spmv_driver.cpp:43-50 pattern):
// returns h2d_count, d2h_count, h2d_bytes, d2h_bytes of one emitted call.
extern "C" int ref_spmv_transfer_probe(int64_t* out4) {
  LAPIS::resetTransferStats();
  LAPIS::DualView<int64_t*> rowptr("rowptr", 5), colind("colind", 5);
  LAPIS::DualView<double*> values("values", 5), x("x", 4), y("y", 4);
  const int64_t rp[5] = {0, 2, 3, 3, 5}, ci[5] = {0, 1, 2, 0, 3};
  const double vv[5] = {1, 2, 3, 4, 5}, xx[4] = {1, 1, 1, 1}, yy[4] = {0, 0, 0, 0};
  fill1(rowptr, rp, 5); fill1(colind, ci, 5); fill1(values, vv, 5);
  fill1(x, xx, 4); fill1(y, yy, 4);
  auto r = spmv(rowptr, colind, values, x, y);
  r.syncHost();
  const auto& s = LAPIS::transferStats();
  out4[0] = (int64_t)s.h2d_count; out4[1] = (int64_t)s.d2h_count;
  out4[2] = (int64_t)s.h2d_bytes; out4[3] = (int64_t)s.d2h_bytes;
  return 0;
}
#endif
