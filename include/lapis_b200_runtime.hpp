// lapis_b200_runtime.hpp — the LAPIS kernel-library seam on the B200 kernels.
//
// The reference emits `LAPIS::gemm(A, B, C)` / `LAPIS::gemv(A, x, y)` for
// kokkos.gemm / kokkos.gemv (emitter.py:550-557) and syncs the operands around
// the call (A, B syncDevice before, C modifyDevice after).  Its runtime header
// implements them as generic templates (runtime_header.py:249-282).  Include
// this header BEFORE the emitted header: its non-template overloads for
// DualView operands win overload resolution, so the unchanged emitted code
// calls the tuned kernels behind include/lapis_b200.h (certified Ozaki / DMMA /
// 3xTF32 GEMM, reference-order GEMV).  It also adds the sparse siblings
// SURVEY 8(b) asks for: LAPIS::spmv_csr and LAPIS::spmm_csr on DualViews.
//
//   nvcc ... --extended-lambda -I include -I include/kokkos_b200 -I <emitted> driver.cpp \
//        -L paper_2509_25605_b200/lib -llapis_b200
//
// All calls run on the legacy default stream (the stream the Kokkos subset in
// include/kokkos_b200 launches on), so they are ordered with the emitted
// kernels; errors abort through Kokkos::abort, as the reference's own runtime.
#pragma once

#include <cstdint>
#include <mutex>
#include <type_traits>
#include <utility>
#include <vector>

#include "lapis_b200.h"
#include "lapis_dualview_runtime.hpp"

namespace LAPIS {
namespace b200 {
template <class T> struct Dtype;
template <> struct Dtype<double> { static constexpr int value = LAPIS_B200_F64; };
template <> struct Dtype<float> { static constexpr int value = LAPIS_B200_F32; };
template <> struct Dtype<std::int64_t> { static constexpr int value = LAPIS_B200_I64; };
template <> struct Dtype<std::int32_t> { static constexpr int value = LAPIS_B200_I32; };

inline void check(int rc) {
  if (rc != LAPIS_B200_OK) Kokkos::abort(lapis_b200_last_error());
}
template <class V>
inline std::int64_t pitch(const V& v) {
  if (v.extent(1) > 1 && v.stride(1) != 1) Kokkos::abort("LAPIS B200 seam: inner stride must be 1");
  return static_cast<std::int64_t>(v.stride(0));
}
template <class V>
inline int index_bytes(const V&) {
  return static_cast<int>(sizeof(typename V::value_type));
}

// Structure plans of LAPIS::spmv_csr, keyed on the identity of rowptr's device
// allocation (View::alloc_id: unique, never reused) and the shape.  A call
// whose rowptr DualView carries a pending host or device modification drops
// the entry and takes the no-plan call (one structure pass on the device);
// the next unmodified call builds a reference-order (exact) plan — one
// analysis read — and every later call replays it.  At most 16 entries, the
// least recently used destroyed first.
template <class V, class = void>
struct HasAllocId : std::false_type {};
template <class V>
struct HasAllocId<V, decltype((void)std::declval<const V&>().alloc_id())> : std::true_type {};

struct CsrPlanCache {
  struct Entry {
    std::uint64_t id;
    const void* rowptr;
    std::int64_t nrows, nnz;
    int rp_bytes;
    lapis_b200_csr_plan plan;
    std::uint64_t used;
  };
  std::mutex mu;
  std::vector<Entry> entries;
  std::uint64_t tick = 0;

  void drop(std::uint64_t id) {
    for (std::size_t i = 0; i < entries.size(); ++i)
      if (entries[i].id == id) {
        lapis_b200_csr_plan_destroy(entries[i].plan);
        entries.erase(entries.begin() + static_cast<std::ptrdiff_t>(i));
        return;
      }
  }
  // the plan for this structure, built on a miss; nullptr when creation fails
  lapis_b200_csr_plan get(std::uint64_t id, const void* rowptr, std::int64_t nrows,
                          std::int64_t nnz, int rp_bytes) {
    for (auto& e : entries)
      if (e.id == id && e.rowptr == rowptr && e.nrows == nrows && e.nnz == nnz &&
          e.rp_bytes == rp_bytes) {
        e.used = ++tick;
        return e.plan;
      }
    drop(id);
    lapis_b200_csr_plan p = nullptr;
    if (lapis_b200_csr_plan_create(nrows, nnz, rowptr, rp_bytes, nullptr, &p) != LAPIS_B200_OK)
      return nullptr;
    if (lapis_b200_csr_plan_set_exact(p, 1) != LAPIS_B200_OK) {
      lapis_b200_csr_plan_destroy(p);
      return nullptr;
    }
    if (entries.size() >= 16) {
      std::size_t lru = 0;
      for (std::size_t i = 1; i < entries.size(); ++i)
        if (entries[i].used < entries[lru].used) lru = i;
      lapis_b200_csr_plan_destroy(entries[lru].plan);
      entries.erase(entries.begin() + static_cast<std::ptrdiff_t>(lru));
    }
    entries.push_back(Entry{id, rowptr, nrows, nnz, rp_bytes, p, ++tick});
    return p;
  }
};
inline CsrPlanCache& csr_plan_cache() {
  static CsrPlanCache* c = new CsrPlanCache();  // never destroyed: plans outlive static teardown
  return *c;
}
inline std::size_t csr_plan_cache_size() {
  std::lock_guard<std::mutex> g(csr_plan_cache().mu);
  return csr_plan_cache().entries.size();
}
}  // namespace b200

// C = A * B on the device copies (runtime_header.py:249-266)
template <class T, class = typename std::enable_if<(b200::Dtype<T>::value >= 0)>::type>
inline void gemm(const DualView<T**>& A, const DualView<T**>& B, const DualView<T**>& C) {
  auto a = A.device_view();
  auto b = B.device_view();
  auto c = C.device_view();
  b200::check(lapis_b200_gemm(static_cast<std::int64_t>(a.extent(0)),
                              static_cast<std::int64_t>(b.extent(1)),
                              static_cast<std::int64_t>(a.extent(1)), a.data(), b200::pitch(a),
                              b.data(), b200::pitch(b), c.data(), b200::pitch(c),
                              b200::Dtype<T>::value, LAPIS_B200_GEMM_AUTO, nullptr));
}
inline void gemm(const DualView<double**>& A, const DualView<double**>& B,
                 const DualView<double**>& C) { gemm<double>(A, B, C); }
inline void gemm(const DualView<float**>& A, const DualView<float**>& B,
                 const DualView<float**>& C) { gemm<float>(A, B, C); }
inline void gemm(const DualView<std::int64_t**>& A, const DualView<std::int64_t**>& B,
                 const DualView<std::int64_t**>& C) { gemm<std::int64_t>(A, B, C); }
inline void gemm(const DualView<std::int32_t**>& A, const DualView<std::int32_t**>& B,
                 const DualView<std::int32_t**>& C) { gemm<std::int32_t>(A, B, C); }

// y = A * x on the device copies (runtime_header.py:268-282)
template <class T, class = typename std::enable_if<(b200::Dtype<T>::value >= 0)>::type>
inline void gemv(const DualView<T**>& A, const DualView<T*>& X, const DualView<T*>& Y) {
  auto a = A.device_view();
  auto x = X.device_view();
  auto y = Y.device_view();
  b200::check(lapis_b200_gemv(static_cast<std::int64_t>(a.extent(0)),
                              static_cast<std::int64_t>(a.extent(1)), a.data(), b200::pitch(a),
                              x.data(), y.data(), b200::Dtype<T>::value, nullptr));
}
inline void gemv(const DualView<double**>& A, const DualView<double*>& X,
                 const DualView<double*>& Y) { gemv<double>(A, X, Y); }
inline void gemv(const DualView<float**>& A, const DualView<float*>& X,
                 const DualView<float*>& Y) { gemv<float>(A, X, Y); }
inline void gemv(const DualView<std::int64_t**>& A, const DualView<std::int64_t*>& X,
                 const DualView<std::int64_t*>& Y) { gemv<std::int64_t>(A, X, Y); }
inline void gemv(const DualView<std::int32_t**>& A, const DualView<std::int32_t*>& X,
                 const DualView<std::int32_t*>& Y) { gemv<std::int32_t>(A, X, Y); }

// y = A x for CSR A: the emitted spmv()'s contract (golden cpp/spmv.hpp:16-70,
// interp.py:798-812) as a library call; syncs the inputs, marks y modified.
template <class RP, class CI, class T>
inline void spmv_csr(DualView<RP*> rowptr, DualView<CI*> colind, DualView<T*> values,
                     DualView<T*> x, DualView<T*> y) {
  // a structure modified since the last call invalidates its cached plan
  const bool rp_modified = rowptr.hostModified() || rowptr.deviceModified();
  rowptr.syncDevice();
  colind.syncDevice();
  values.syncDevice();
  x.syncDevice();
  const std::int64_t n = rowptr.extent(0) - 1;
  // nnz bound from colind's extent (>= rowptr(n) - rowptr(0) for any valid
  // CSR): no read of a host copy that may be stale after a device write
  const std::int64_t nnz = static_cast<std::int64_t>(colind.extent(0));
  auto rp = rowptr.device_view();
  auto ci = colind.device_view();
  lapis_b200_csr_plan plan = nullptr;
  if constexpr (b200::HasAllocId<decltype(rp)>::value) {
    const std::uint64_t id = rp.alloc_id();
    if (id != 0 && n > 0 && rp.stride(0) == 1) {
      auto& cache = b200::csr_plan_cache();
      std::lock_guard<std::mutex> g(cache.mu);
      if (rp_modified)
        cache.drop(id);
      else
        plan = cache.get(id, rp.data(), n, nnz, b200::index_bytes(rp));
    }
  }
  if (plan)
    b200::check(lapis_b200_spmv_csr_plan(plan, rp.data(), b200::index_bytes(rp), ci.data(),
                                         b200::index_bytes(ci), values.device_view().data(),
                                         x.device_view().data(), y.device_view().data(),
                                         b200::Dtype<T>::value, nullptr));
  else
    b200::check(lapis_b200_spmv_csr(n, x.extent(0), nnz, rp.data(), b200::index_bytes(rp),
                                    ci.data(), b200::index_bytes(ci), values.device_view().data(),
                                    x.device_view().data(), y.device_view().data(),
                                    b200::Dtype<T>::value, 0, nullptr));
  y.modifyDevice();
}

// Y = A X for CSR A and row-major X [ncols, k] (oracle/ir/spmm.mlir)
template <class RP, class CI, class T>
inline void spmm_csr(DualView<RP*> rowptr, DualView<CI*> colind, DualView<T*> values,
                     DualView<T**> X, DualView<T**> Y) {
  rowptr.syncDevice();
  colind.syncDevice();
  values.syncDevice();
  X.syncDevice();
  const std::int64_t n = rowptr.extent(0) - 1;
  const std::int64_t nnz = static_cast<std::int64_t>(colind.extent(0));  // as in spmv_csr
  auto rp = rowptr.device_view();
  auto ci = colind.device_view();
  auto xd = X.device_view();
  auto yd = Y.device_view();
  b200::check(lapis_b200_spmm_csr(n, X.extent(0), nnz, X.extent(1), rp.data(), b200::index_bytes(rp),
                                  ci.data(), b200::index_bytes(ci), values.device_view().data(),
                                  xd.data(), b200::pitch(xd), yd.data(), b200::pitch(yd),
                                  b200::Dtype<T>::value, nullptr));
  Y.modifyDevice();
}

}  // namespace LAPIS
