// common.cuh — shared helpers for the sm_100a kernels behind include/lapis_b200.h.
#pragma once

#include <nvtx3/nvToolsExt.h>

#include <cstdlib>
#include <cstring>

#include <cuda_runtime.h>
#include <cstdint>
#include <string>

#include "../../include/lapis_b200.h"

namespace lapis_b200 {

// NVTX range around each C-ABI entry point (visible in nsys / ncu --nvtx;
// header-only NVTX v3: a no-op unless a tool injects itself)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define LB_RANGE(name) ::lapis_b200::NvtxRange lb_nvtx_range_(name)

// ------------------------------------------------------------------ errors
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int check_cuda(cudaError_t e, const char* what);
int check_launch(const char* what);

#define LB_TRY(expr)              \
  do {                            \
    int _rc = (expr);             \
    if (_rc != LAPIS_B200_OK) return _rc; \
  } while (0)

// ------------------------------------------------------- element arithmetic
// Reference semantics: every op is rounded to the element type before the next
// one (interp.py:168-183), ints wrap (interp.py:145-152).  The explicit _rn
// intrinsics keep nvcc from contracting mul+add into an FMA, so a sequential
// sum reproduces the reference bit for bit.
template <class T> struct Arith;
template <> struct Arith<double> {
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double zero() { return 0.0; }
};
template <> struct Arith<float> {
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float zero() { return 0.0f; }
};
template <> struct Arith<long long> {
  static __device__ __forceinline__ long long mul(long long a, long long b) {
    return (long long)((unsigned long long)a * (unsigned long long)b);
  }
  static __device__ __forceinline__ long long add(long long a, long long b) {
    return (long long)((unsigned long long)a + (unsigned long long)b);
  }
  static __device__ __forceinline__ long long zero() { return 0; }
};
template <> struct Arith<int> {
  static __device__ __forceinline__ int mul(int a, int b) { return (int)((unsigned)a * (unsigned)b); }
  static __device__ __forceinline__ int add(int a, int b) { return (int)((unsigned)a + (unsigned)b); }
  static __device__ __forceinline__ int zero() { return 0; }
};

// warp shuffle for 64-bit types
template <class T>
__device__ __forceinline__ T shfl_xor(T v, int mask, int width = 32) {
  return __shfl_xor_sync(0xffffffffu, v, mask, width);
}

// streaming (read-once) loads: bypass L1 allocation, keep L2 policy default
__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
               : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ longlong2 ld_stream(const longlong2* p) {
  longlong2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.s64 {%0,%1}, [%2];"
               : "=l"(r.x), "=l"(r.y) : "l"(p));
  return r;
}

// Stream-ordered scratch (cudaMallocAsync) comes from the device's default
// memory pool; keep freed blocks cached in the pool instead of returning them
// to the driver at every synchronisation (the default release threshold of 0
// turns every per-call workspace into a fresh mapping).
inline void keep_pool_memory() {
  static bool done[64] = {false};
  static const bool off = [] {
    const char* e = getenv("LAPIS_B200_KEEP_POOL");
    return e && e[0] == '0';
  }();
  if (off) return;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev] = true;
}

// Device-side launch guard: a fallback kernel launched unconditionally that
// returns at once unless its flag condition holds (keeps data-dependent
// fallbacks stream-ordered, no host sync).  mode 0: always run; mode 1: run
// iff flags[0]; mode 2: run iff !flags[0] && flags[1].
struct Guard {
  const int* flags = nullptr;
  int mode = 0;
};
__device__ __forceinline__ bool guard_skip(const Guard& g) {
  if (g.mode == 0 || !g.flags) return false;
  if (g.mode == 1) return g.flags[0] == 0;
  return g.flags[0] != 0 || g.flags[1] == 0;
}

// GEMM paths shared across translation units (dense.cu dispatches; the Ozaki
// path launches the others as guarded fallbacks)
int gemm_tf32x3(int64_t batch, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda,
                const void* B, int64_t ldb, void* C, int64_t ldc, int64_t sA, int64_t sB,
                int64_t sC, cudaStream_t st, Guard guard = Guard());
int gemm_dmma(int64_t batch, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda,
              const void* B, int64_t ldb, void* C, int64_t ldc, int64_t sA, int64_t sB,
              int64_t sC, cudaStream_t st, Guard guard = Guard());
int launch_gemm_exact_guarded(int64_t m, int64_t n, int64_t k, const void* A, int64_t lda,
                              const void* B, int64_t ldb, void* C, int64_t ldc, int dtype,
                              Guard guard, cudaStream_t st);

inline int elem_bytes(int dtype) {
  return (dtype == LAPIS_B200_F64 || dtype == LAPIS_B200_I64) ? 8 : 4;
}
inline bool valid_dtype(int dtype) { return dtype >= LAPIS_B200_F32 && dtype <= LAPIS_B200_I64; }

inline int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (!cached[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = v > 0 ? v : 148;
  }
  return cached[dev];
}

// A per-device, highest-priority, non-blocking stream for work that may run
// concurrently with the caller's stream inside one library call (forked and
// joined with events, so the call stays stream-ordered for the caller and is
// graph-capturable).  nullptr when it cannot be created (the caller then
// stays on its own stream).  LAPIS_B200_NO_SIDE_STREAM=1 disables it.
inline cudaStream_t long_row_stream() {
  static cudaStream_t streams[64] = {nullptr};
  static int disabled = -1;
  if (disabled < 0) {
    const char* e = getenv("LAPIS_B200_NO_SIDE_STREAM");
    disabled = (e && e[0] == '1') ? 1 : 0;
  }
  if (disabled) return nullptr;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  if (!streams[dev]) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStream_t s = nullptr;
    if (cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, hi) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    streams[dev] = s;
  }
  return streams[dev];
}

}  // namespace lapis_b200

// ------------------------------------------------------ async-proxy helpers
// mbarrier + TMA bulk copy (cp.async.bulk) primitives, sm_90+ / sm_100a PTX.
namespace lapis_b200 {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, p;\n\t}"
        : "=r"(done) : "r"(addr), "r"(parity) : "memory");
  } while (!done);
}
// 1-D bulk copy global -> shared (TMA engine), completion counted on `bar`.
// dst, src 16-byte aligned; bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

}  // namespace lapis_b200

// ------------------------------------------------------ L2 cache-policy loads
// Streams read once (colind, values) are loaded with an L2 evict_first policy so
// they do not push out data with reuse (the gathered x); gathers use evict_last.
namespace lapis_b200 {

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Ordered read-only loads: asm volatile statements keep their program order,
// so a batch of these is ISSUED in the order written (all index loads of a
// batch, then all gathers) instead of being interleaved by the scheduler with
// the loads that depend on them; a predicated-off load returns 0.
template <class T> __device__ __forceinline__ T ld_ord(const T* p, bool pred);
template <> __device__ __forceinline__ double ld_ord<double>(const double* p, bool pred) {
  double v;
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\tmov.f64 %0, 0d0000000000000000;\n\t"
               "@q ld.global.nc.f64 %0, [%1];\n\t}" : "=d"(v) : "l"(p), "r"((int)pred));
  return v;
}
template <> __device__ __forceinline__ float ld_ord<float>(const float* p, bool pred) {
  float v;
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\tmov.f32 %0, 0f00000000;\n\t"
               "@q ld.global.nc.f32 %0, [%1];\n\t}" : "=f"(v) : "l"(p), "r"((int)pred));
  return v;
}
template <> __device__ __forceinline__ long long ld_ord<long long>(const long long* p, bool pred) {
  long long v;
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\tmov.b64 %0, 0;\n\t"
               "@q ld.global.nc.b64 %0, [%1];\n\t}" : "=l"(v) : "l"(p), "r"((int)pred));
  return v;
}
template <> __device__ __forceinline__ long ld_ord<long>(const long* p, bool pred) {
  return (long)ld_ord<long long>(reinterpret_cast<const long long*>(p), pred);
}
template <> __device__ __forceinline__ int ld_ord<int>(const int* p, bool pred) {
  int v;
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\tmov.b32 %0, 0;\n\t"
               "@q ld.global.nc.b32 %0, [%1];\n\t}" : "=r"(v) : "l"(p), "r"((int)pred));
  return v;
}

template <class T> __device__ __forceinline__ T ld_hint(const T* p, uint64_t pol);
template <> __device__ __forceinline__ double ld_hint<double>(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
template <> __device__ __forceinline__ float ld_hint<float>(const float* p, uint64_t pol) {
  float v;
  asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
template <> __device__ __forceinline__ long long ld_hint<long long>(const long long* p, uint64_t pol) {
  long long v;
  asm volatile("ld.global.nc.L2::cache_hint.s64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  return v;
}
template <> __device__ __forceinline__ int ld_hint<int>(const int* p, uint64_t pol) {
  int v;
  asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
template <> __device__ __forceinline__ long ld_hint<long>(const long* p, uint64_t pol) {
  long v;
  asm volatile("ld.global.nc.L2::cache_hint.s64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  return v;
}

}  // namespace lapis_b200
