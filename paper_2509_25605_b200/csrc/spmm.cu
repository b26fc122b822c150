// spmm.cu — CSR x dense SpMM for sm_100a:  Y[i, c] = sum_j values[j] * X[colind[j], c].
//
// The reference has no SpMM op; the loop nest oracle/ir/spmm.mlir
// is what its preset lowers (thread_parallel over N*K, CSR vector-length hint),
// with the per-(i, c) order of interp.py:798-812: j ascending, mul and add
// each rounded.
//
// Kernel 1 (spmm_batch_kernel when k is a multiple of 32; spmm_group_kernel /
//   spmm_row_kernel otherwise): every row of <= SPLIT entries, each dense
//   column summed in ascending entry order with non-contracted mul/add ->
//   bit-identical to the reference.
// Long rows (> SPLIT entries; power-law hubs, config 3: 117,686 entries) are
//   listed by one pass over rowptr, then folded in exact order (fp32,
//   spmm_seq_long_pipe_kernel) or cut into SPLIT-entry chunks whose partials a
//   persistent CTA pool computes and a combine kernel adds in chunk order
//   (other types; deterministic, no atomics on values).
#include "common.cuh"

#include <cub/device/device_radix_sort.cuh>

#include <cstdlib>
#include <type_traits>
#include <vector>
#include <algorithm>

namespace lapis_b200 {

constexpr int SPMM_WARPS = 8;
constexpr int64_t SPLIT = 2048;

// A rowptr that decreases somewhere (row r has rowptr[r+1] < rowptr[r]; the
// reference sums range(begin, max(begin, end)), interp.py:808) breaks the
// batch kernel's contiguous entry runs and the long-row list's capacity
// bound.  The long-row list pass flags it on the device (desc[0] != 0); the
// fast kernels then return at once and a one-warp-per-row kernel, launched
// behind the same flag, folds every row (long ones included) on its clamped
// range.  No host round trip: the call stays stream-ordered.
struct DescGuard {
  const unsigned long long* desc = nullptr;  // nullptr: unguarded
  int mode = 0;  // 0: run unless desc set; 1: run only when desc set (all rows)
  __device__ __forceinline__ bool skip() const {
    if (!desc) return false;
    return (*(volatile const unsigned long long*)desc != 0) != (mode == 1);
  }
  __device__ __forceinline__ bool all_rows() const { return desc && mode == 1; }
};

// --------------------------------------------------------------- kernel 1
template <class T, class RP, class CI, int EPL>
__global__ void __launch_bounds__(SPMM_WARPS * 32)
spmm_row_kernel(int64_t nrows, int64_t k, const RP* __restrict__ rowptr,
                const CI* __restrict__ colind, const T* __restrict__ values,
                const T* __restrict__ X, int64_t ldx, T* __restrict__ Y, int64_t ldy,
                DescGuard guard = DescGuard()) {
  if (guard.skip()) return;
  const int lane = threadIdx.x & 31;
  // grid-stride over rows, one warp per row (a guarded launch that is not
  // selected costs one small grid, not one CTA per 8 rows)
  for (int64_t row = (int64_t)blockIdx.x * SPMM_WARPS + (threadIdx.x >> 5); row < nrows;
       row += (int64_t)gridDim.x * SPMM_WARPS) {
  const int64_t b = (int64_t)rowptr[row];
  int64_t e = (int64_t)rowptr[row + 1];
  if (e < b) e = b;
  if (e - b > SPLIT && !guard.all_rows()) continue;  // long row: kernels 2-3
  for (int64_t c0 = 0; c0 < k; c0 += 32 * EPL) {
    const int64_t col = c0 + (int64_t)lane * EPL;
    const bool full = col + EPL <= k;
    T acc[EPL];
#pragma unroll
    for (int q = 0; q < EPL; ++q) acc[q] = Arith<T>::zero();
    int64_t j = b;
    for (; j + 4 <= e; j += 4) {
      T v[4];
      int64_t ci[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { v[u] = values[j + u]; ci[u] = (int64_t)colind[j + u]; }
      T xv[4][EPL];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const T* xr = X + ci[u] * ldx + col;
        if (EPL == 2 && full) {
          if constexpr (sizeof(T) == 8) {
            const longlong2 w = __ldg(reinterpret_cast<const longlong2*>(xr));
            memcpy(&xv[u][0], &w.x, 8);
            memcpy(&xv[u][EPL - 1], &w.y, 8);
          } else {
            const int2 w = __ldg(reinterpret_cast<const int2*>(xr));
            memcpy(&xv[u][0], &w.x, 4);
            memcpy(&xv[u][EPL - 1], &w.y, 4);
          }
        } else {
#pragma unroll
          for (int q = 0; q < EPL; ++q) xv[u][q] = (col + q < k) ? __ldg(xr + q) : Arith<T>::zero();
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int q = 0; q < EPL; ++q) acc[q] = Arith<T>::add(acc[q], Arith<T>::mul(v[u], xv[u][q]));
    }
    for (; j < e; ++j) {
      const T v = values[j];
      const T* xr = X + (int64_t)colind[j] * ldx + col;
#pragma unroll
      for (int q = 0; q < EPL; ++q)
        if (col + q < k) acc[q] = Arith<T>::add(acc[q], Arith<T>::mul(v, __ldg(xr + q)));
    }
    T* yr = Y + row * ldy + col;
#pragma unroll
    for (int q = 0; q < EPL; ++q)
      if (col + q < k) yr[q] = acc[q];
  }
  }
}

// ------------------------------------------------------ kernel 1 (grouped)
// G lanes per row, 4 consecutive dense columns per lane (fp64: two 16-byte
// gathers per X row slice), 32/G rows per warp, persistent grid-stride over
// row groups.  The entries of a row are walked 4 at a time with predication:
// out-of-row steps contribute value 0 * x 0 = +0.0, which leaves the running
// per-column sum unchanged, so the ascending sequential order (and the
// bit-identity with the reference) is kept while 4 X-row gathers per row are
// in flight.
template <class T>
__device__ __forceinline__ void ldg4(const T* p, T (&v)[4]) {
  if constexpr (sizeof(T) == 8) {
    const longlong2 a = __ldg(reinterpret_cast<const longlong2*>(p));
    const longlong2 b = __ldg(reinterpret_cast<const longlong2*>(p + 2));
    memcpy(&v[0], &a.x, 8); memcpy(&v[1], &a.y, 8); memcpy(&v[2], &b.x, 8); memcpy(&v[3], &b.y, 8);
  } else {
    const int4 a = __ldg(reinterpret_cast<const int4*>(p));
    memcpy(&v[0], &a.x, 4); memcpy(&v[1], &a.y, 4); memcpy(&v[2], &a.z, 4); memcpy(&v[3], &a.w, 4);
  }
}
template <class T>
__device__ __forceinline__ void stg4(T* p, const T (&v)[4]) {
  if constexpr (sizeof(T) == 8) {
    longlong2 a, b;
    memcpy(&a.x, &v[0], 8); memcpy(&a.y, &v[1], 8); memcpy(&b.x, &v[2], 8); memcpy(&b.y, &v[3], 8);
    *reinterpret_cast<longlong2*>(p) = a;
    *reinterpret_cast<longlong2*>(p + 2) = b;
  } else {
    int4 a;
    memcpy(&a.x, &v[0], 4); memcpy(&a.y, &v[1], 4); memcpy(&a.z, &v[2], 4); memcpy(&a.w, &v[3], 4);
    *reinterpret_cast<int4*>(p) = a;
  }
}

template <class T, class RP, class CI, int G>
__global__ void __launch_bounds__(256)
spmm_group_kernel(int64_t nrows, int64_t k, const RP* __restrict__ rowptr,
                  const CI* __restrict__ colind, const T* __restrict__ values,
                  const T* __restrict__ X, int64_t ldx, T* __restrict__ Y, int64_t ldy,
                  DescGuard guard = DescGuard()) {
  if (guard.skip()) return;
  constexpr int U = 4;
  const int lane = threadIdx.x & (G - 1);
  const int64_t groups = (int64_t)gridDim.x * (blockDim.x / G);
  const int64_t g0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  for (int64_t row = g0; row < nrows; row += groups) {
    const int64_t b = (int64_t)rowptr[row];
    int64_t e = (int64_t)rowptr[row + 1];
    if (e < b) e = b;
    if (e - b > SPLIT) continue;  // long row: kernels 2-3
    for (int64_t c0 = 4 * lane; c0 < k; c0 += 4 * G) {
      T acc[4] = {Arith<T>::zero(), Arith<T>::zero(), Arith<T>::zero(), Arith<T>::zero()};
      for (int64_t j0 = b; j0 < e; j0 += U) {
        T v[U];
        int64_t ci[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const bool ok = j0 + u < e;
          v[u] = ok ? values[j0 + u] : T(0);
          ci[u] = ok ? (int64_t)colind[j0 + u] : -1;
        }
        T xv[U][4];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (ci[u] >= 0) {
            ldg4(X + ci[u] * ldx + c0, xv[u]);
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) xv[u][q] = T(0);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[q] = Arith<T>::add(acc[q], Arith<T>::mul(v[u], xv[u][q]));
      }
      T* yr = Y + row * ldy + c0;
      stg4(yr, acc);
    }
  }
}

// ------------------------------------------------------ kernel 1 (batched)
// A warp owns a batch of 32 consecutive rows.  Lane l holds rowptr[r0 + l],
// so the row structure of the batch costs one coalesced load; colind/values
// are read 32 entries at a time (coalesced, the next chunk prefetched while the
// current one is consumed) and broadcast by shuffles; X-row gathers are issued
// U entries ahead ACROSS row boundaries, so the memory pipeline never waits on
// a per-row dependency chain (rowptr -> colind -> X) — the limiter of the
// one-row-per-warp kernel on short power-law rows (median 5 entries).  Each
// lane owns CPL consecutive dense columns; every column is still summed in
// ascending entry order with non-contracted mul / add (bit-identical).  A
// batch holding a row longer than SPLIT walks its rows one by one and leaves
// the long rows to kernels 2-3.
template <class T, int CPL>
struct XVec;
template <> struct XVec<double, 1> { using V = double; };
template <> struct XVec<double, 2> { using V = longlong2; };
template <> struct XVec<double, 4> { using V = longlong4; };
template <> struct XVec<float, 1> { using V = float; };
template <> struct XVec<float, 2> { using V = int2; };
template <> struct XVec<float, 4> { using V = int4; };
template <> struct XVec<long long, 1> { using V = long long; };
template <> struct XVec<long long, 2> { using V = longlong2; };
template <> struct XVec<long long, 4> { using V = longlong4; };
template <> struct XVec<int, 1> { using V = int; };
template <> struct XVec<int, 2> { using V = int2; };
template <> struct XVec<int, 4> { using V = int4; };

template <class T, int CPL>
__device__ __forceinline__ void ldx_row(const T* p, T (&v)[CPL]) {
  using V = typename XVec<T, CPL>::V;
  const V w = *reinterpret_cast<const V*>(p);
  memcpy(&v[0], &w, sizeof(V));
}
template <class T, int CPL>
__device__ __forceinline__ void sty_row(T* p, const T (&v)[CPL]) {
  using V = typename XVec<T, CPL>::V;
  V w;
  memcpy(&w, &v[0], sizeof(V));
  *reinterpret_cast<V*>(p) = w;
}

// X-row slice load with an L2 eviction-priority policy (SpMM plans with reuse
// hints): one instruction whatever the policy, so lanes of a warp may carry
// different policies
template <class T, int CPL>
__device__ __forceinline__ void ldx_row_pol(const T* p, T (&v)[CPL], uint64_t pol) {
  using V = typename XVec<T, CPL>::V;
  if constexpr (sizeof(V) == 4) {
    uint32_t w;
    asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(w) : "l"(p), "l"(pol));
    memcpy(&v[0], &w, 4);
  } else if constexpr (sizeof(V) == 8) {
    unsigned long long w;
    asm volatile("ld.global.nc.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(w) : "l"(p), "l"(pol));
    memcpy(&v[0], &w, 8);
  } else {
    static_assert(sizeof(V) % 16 == 0, "ldx_row_pol: 4, 8, 16 or 32 bytes");
#pragma unroll
    for (int h = 0; h < (int)(sizeof(V) / 16); ++h) {
      unsigned long long a, b;
      asm volatile("ld.global.nc.L2::cache_hint.v2.b64 {%0,%1}, [%2], %3;"
                   : "=l"(a), "=l"(b) : "l"(reinterpret_cast<const char*>(p) + 16 * h), "l"(pol));
      memcpy(reinterpret_cast<char*>(&v[0]) + 16 * h, &a, 8);
      memcpy(reinterpret_cast<char*>(&v[0]) + 16 * h + 8, &b, 8);
    }
  }
}
// bit 30 of a non-negative remapped column: the X row's next use lies beyond
// the plan's reuse horizon (loaded L2::evict_first)
constexpr int32_t SPMM_FAR_BIT = 1 << 30;

// ------------------------------------------------ fused GCN epilogue (fp32)
// H[row, :] = relu(AX[row, :] W) for one row held by the warp as 2 values per
// lane (lane l: AX[row, 2l], AX[row, 2l+1]; fin = fout = 64), W staged in shared
// memory.  The reference order of the GCN's linalg.matmul (oracle/ir/gcn_f32.mlir,
// interp.py:711-722): k ascending from 0.0f, mul and add each rounded — the same
// arithmetic as gemm_exact_narrow_kernel — then the cmpf ogt + select ReLU.
// Not inlined: it is called from every row-end point of the unrolled batch loop.
constexpr int GCN_F = 64;
__device__ __noinline__ void gcn_row_epilogue(float a0, float a1, const float* __restrict__ Ws,
                                              float* __restrict__ hrow, int lane) {
  float o0 = 0.0f, o1 = 0.0f;
  const float2* w2 = reinterpret_cast<const float2*>(Ws) + lane;
#pragma unroll 8
  for (int kb = 0; kb < 32; ++kb) {
    const float x0 = __shfl_sync(0xffffffffu, a0, kb);
    const float x1 = __shfl_sync(0xffffffffu, a1, kb);
    const float2 b0 = w2[(2 * kb) * (GCN_F / 2)];
    const float2 b1 = w2[(2 * kb + 1) * (GCN_F / 2)];
    o0 = __fadd_rn(o0, __fmul_rn(x0, b0.x));
    o1 = __fadd_rn(o1, __fmul_rn(x0, b0.y));
    o0 = __fadd_rn(o0, __fmul_rn(x1, b1.x));
    o1 = __fadd_rn(o1, __fmul_rn(x1, b1.y));
  }
  float2 h;
  h.x = (o0 > 0.0f) ? o0 : 0.0f;
  h.y = (o1 > 0.0f) ? o1 : 0.0f;
  reinterpret_cast<float2*>(hrow)[lane] = h;
}

// L2 prefetch of the next gather group (kernel argument `pf`, default 1;
// LAPIS_B200_SPMM_PREFETCH=0 disables, N = gather groups ahead; 1 measured
// best: C3 10.05 / 11.6 / 13.8 ms at 1 / 2 / 3, C4 1.64 -> 1.55 ms at 1)
inline int spmm_prefetch_distance() {
  static const int pf = [] {
    const char* e = getenv("LAPIS_B200_SPMM_PREFETCH");
    int v = e ? atoi(e) : 1;
    return v < 0 ? 0 : (v > 4 ? 4 : v);
  }();
  return pf;
}

template <class T, class RP, class CI, int CPL, int U, bool EPI = false>
__global__ void __launch_bounds__(256, 4)
spmm_batch_kernel(int64_t nrows, int64_t k, const RP* __restrict__ rowptr,
                  const CI* __restrict__ colind, const T* __restrict__ values,
                  const T* __restrict__ X, int64_t ldx, T* __restrict__ Y, int64_t ldy,
                  const T* __restrict__ W = nullptr,
                  unsigned long long* __restrict__ next = nullptr, int pf = 1,
                  DescGuard guard = DescGuard()) {
  if (guard.skip()) return;
  const int lane = threadIdx.x & 31;
  // EPI (fp32, k = 64, CPL = 2): Y is H, each finished row goes through the
  // GCN epilogue with W staged in shared memory
  __shared__ __align__(16) float Ws[EPI ? GCN_F * GCN_F : 1];
  if constexpr (EPI) {
    for (int t = threadIdx.x; t < GCN_F * GCN_F; t += blockDim.x) Ws[t] = W[t];
    __syncthreads();
  }
  auto store_row = [&](int64_t row, const T (&a)[CPL], int64_t c0) {
    if constexpr (EPI) {
      static_assert(CPL == 2, "GCN epilogue: fin = 64");
      gcn_row_epilogue(a[0], a[1], Ws, Y + row * ldy, lane);
    } else {
      sty_row<T, CPL>(Y + row * ldy + c0, a);
    }
  };
  const int64_t nbatch = (nrows + 31) >> 5;
  const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // batches of 32 rows are handed out one at a time from a global counter
  // (`next`, zeroed per call): row lengths vary by orders of magnitude, and a
  // static grid-stride split leaves SMs with finished warps that cannot take
  // a new CTA until the slowest warp of theirs is done
  auto grab = [&]() -> int64_t {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(next, 1ull);
    return (int64_t)__shfl_sync(0xffffffffu, t, 0);
  };
  for (int64_t bt = next ? grab() : (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
       bt < nbatch; bt = next ? grab() : bt + wstride) {
    const int64_t r0 = bt << 5;
    const int nr = (int)((nrows - r0) < 32 ? (nrows - r0) : 32);
    const int64_t rp_l = (int64_t)rowptr[r0 + (lane < nr ? lane : nr)];
    const int64_t rp_end = (int64_t)rowptr[r0 + nr];   // one broadcast load
    // row lengths (monotone rowptr is validated by the executor)
    const int64_t dn = __shfl_down_sync(0xffffffffu, rp_l, 1);
    const int64_t nxt_l = (lane + 1 < nr) ? dn : rp_end;
    // rows longer than SPLIT are left to the long-row kernels: the batch is
    // walked as maximal runs of short rows [ra, rb), each run one contiguous
    // entry range
    const unsigned long_mask = __ballot_sync(0xffffffffu, lane < nr && (nxt_l - rp_l) > SPLIT);
    for (int64_t c0 = (int64_t)lane * CPL; c0 - (int64_t)lane * CPL < k; c0 += 32 * CPL) {
      int ra = 0;
      while (ra < nr) {
        if ((long_mask >> ra) & 1u) { ++ra; continue; }
        const unsigned above = long_mask & ~((2u << ra) - 1u);   // long rows after ra
        const int rb = above ? (__ffs(above) - 1) : nr;
        const int64_t jb = __shfl_sync(0xffffffffu, rp_l, ra);
        const int64_t je = rb < nr ? __shfl_sync(0xffffffffu, rp_l, rb & 31) : rp_end;
        int cur = ra;
        int64_t nxt = (cur + 1 < nr) ? __shfl_sync(0xffffffffu, rp_l, (cur + 1) & 31) : rp_end;
        T acc[CPL];
#pragma unroll
        for (int q = 0; q < CPL; ++q) acc[q] = Arith<T>::zero();
        int64_t my_col = 0;
        T my_val = T(0);
        if (jb + lane < je) { my_col = (int64_t)colind[jb + lane]; my_val = values[jb + lane]; }
        for (int64_t j0 = jb; j0 < je; j0 += 32) {
          const int cnt = (int)((je - j0) < 32 ? (je - j0) : 32);
          // prefetch the next chunk's structure
          int64_t nx_col = 0;
          T nx_val = T(0);
          if (j0 + 32 + lane < je) { nx_col = (int64_t)colind[j0 + 32 + lane]; nx_val = values[j0 + 32 + lane]; }
          for (int t0 = 0; t0 < cnt; t0 += U) {
            if (pf) {
              // L2 prefetch of the NEXT group's X rows (no registers held): lane
              // l touches line (l / U) of entry t0 + U + l % U; past the chunk
              // end the next chunk's entries (colind already loaded) are used
              const int pe = t0 + U * pf + (lane % U);
              const int64_t pc = pe < 32 ? __shfl_sync(0xffffffffu, my_col, pe & 31)
                                         : __shfl_sync(0xffffffffu, nx_col, pe & 31);
              const int64_t pj = j0 + pe;
              const int line = lane / U;
              if (pj < je && (int64_t)line * (128 / (int64_t)sizeof(T)) < 32 * CPL)
                asm volatile("prefetch.global.L2 [%0];" ::
                             "l"(X + pc * ldx + c0 - lane * CPL + line * (128 / sizeof(T))));
            }
            T xv[U][CPL];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int64_t c = __shfl_sync(0xffffffffu, my_col, (t0 + u) & 31);
              if (t0 + u < cnt) {
                ldx_row<T, CPL>(X + c * ldx + c0, xv[u]);
              } else {
#pragma unroll
                for (int q = 0; q < CPL; ++q) xv[u][q] = T(0);
              }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const T v = __shfl_sync(0xffffffffu, my_val, (t0 + u) & 31);
              if (t0 + u < cnt) {
                const int64_t j = j0 + t0 + u;
                while (j == nxt) {  // rows that end here (empty rows included)
                  store_row(r0 + cur, acc, c0);
#pragma unroll
                  for (int q = 0; q < CPL; ++q) acc[q] = Arith<T>::zero();
                  ++cur;
                  nxt = (cur + 1 < nr) ? __shfl_sync(0xffffffffu, rp_l, (cur + 1) & 31) : rp_end;
                }
#pragma unroll
                for (int q = 0; q < CPL; ++q) acc[q] = Arith<T>::add(acc[q], Arith<T>::mul(v, xv[u][q]));
              }
            }
          }
          my_col = nx_col;
          my_val = nx_val;
        }
        for (; cur < rb; ++cur) {  // the run's last rows (and trailing empty rows)
          store_row(r0 + cur, acc, c0);
#pragma unroll
          for (int q = 0; q < CPL; ++q) acc[q] = Arith<T>::zero();
        }
        ra = rb;
      }
    }
  }
}

// ------------------------------------------------ kernel 1 (batched, lean)
// The batch kernel's algorithm with the per-entry control made provably
// warp-uniform: the batch's 33 row pointers live in shared memory (the
// row-end test reads them with a broadcast load instead of a shuffle), every
// shuffle is executed unconditionally (no collective/convergence fix-ups
// around predicated shuffles), column indices stay in their stored width, and
// the L2 prefetch distance is a template constant.  Same arithmetic, same
// order (bit-identical); ncu on config 4: 53 warp instructions per nonzero
// and 74 % issue-active for the original loop.
// HOT (SpMM plans, lapis_b200_spmm_plan_*): colind is the plan's remapped
// copy — a negative entry ~h addresses row h of Xh, the compact copy of the
// most referenced X rows, which the plan pins in L2 with a persisting access
// policy window; other entries address X as usual.  Entry order unchanged.
// Three CTAs per SM (up to 80 registers): config 3 without a plan 9.91 -> 7.89
// ms, with a plan 8.78 -> 7.61 ms (kernel) against four CTAs per SM
template <class T, class RP, class CI, int CPL, int U, int PF, bool HOT = false>
__global__ void __launch_bounds__(256, (U > 16 ? 2 : 3))
spmm_batch2_kernel(int64_t nrows, int64_t k, const RP* __restrict__ rowptr,
                   const CI* __restrict__ colind, const T* __restrict__ values,
                   const T* __restrict__ X, int64_t ldx, T* __restrict__ Y, int64_t ldy,
                   unsigned long long* __restrict__ next, DescGuard guard,
                   const T* __restrict__ Xh = nullptr, int64_t ldh = 0, int farpf = 0) {
  if (guard.skip()) return;
  __shared__ int64_t s_rp_all[8][33];
  const int lane = threadIdx.x & 31;
  int64_t* s_rp = s_rp_all[threadIdx.x >> 5];
  const int64_t nbatch = (nrows + 31) >> 5;
  // HOT plans with reuse hints: X rows whose next use is far are loaded
  // evict_first (they would only push out rows with reuse), the rest evict_normal
  uint64_t pol_far = 0, pol_near = 0, pol_hot = 0;
  if constexpr (HOT) {
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_far));
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_near));
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_hot));
  }
  for (;;) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(next, 1ull);
    const int64_t bt = (int64_t)__shfl_sync(0xffffffffu, t, 0);
    if (bt >= nbatch) break;
    const int64_t r0 = bt << 5;
    const int nr = (int)((nrows - r0) < 32 ? (nrows - r0) : 32);
    __syncwarp();
    if (lane <= nr) s_rp[lane] = (int64_t)rowptr[r0 + lane];
    if (nr == 32 && lane == 0) s_rp[32] = (int64_t)rowptr[r0 + 32];
    __syncwarp();
    const int64_t my_len = lane < nr ? s_rp[lane + 1] - s_rp[lane] : 0;
    const unsigned long_mask = __ballot_sync(0xffffffffu, my_len > SPLIT);
    for (int64_t c0 = (int64_t)lane * CPL; c0 - (int64_t)lane * CPL < k; c0 += 32 * CPL) {
      // X rows are addressed as base + col * pitch with one 32x32->64-bit
      // multiply-add (column index and pitch in bytes both < 2^32)
      const char* xbase = reinterpret_cast<const char*>(X + c0);
      const uint32_t ldxb = (uint32_t)(ldx * (int64_t)sizeof(T));
      const char* hbase = HOT ? reinterpret_cast<const char*>(Xh + c0) : nullptr;
      const uint32_t ldhb = (uint32_t)(ldh * (int64_t)sizeof(T));
      int ra = 0;
      while (ra < nr) {
        if ((long_mask >> ra) & 1u) { ++ra; continue; }
        const unsigned above = long_mask & ~((2u << ra) - 1u);
        const int rb = above ? (__ffs(above) - 1) : nr;
        const int64_t jb = s_rp[ra], je = s_rp[rb];
        int cur = ra;
        int64_t nxt = s_rp[ra + 1];
        T* yrow = Y + (r0 + ra) * ldy + c0;
        T acc[CPL];
#pragma unroll
        for (int q = 0; q < CPL; ++q) acc[q] = Arith<T>::zero();
        CI my_col = 0;
        T my_val = T(0);
        if (jb + lane < je) { my_col = colind[jb + lane]; my_val = values[jb + lane]; }
        for (int64_t j0 = jb; j0 < je; j0 += 32) {
          const int cnt = (int)((je - j0) < 32 ? (je - j0) : 32);
          CI nx_col = 0;
          T nx_val = T(0);
          if (j0 + 32 + lane < je) { nx_col = colind[j0 + 32 + lane]; nx_val = values[j0 + 32 + lane]; }
          for (int t0 = 0; t0 < cnt; t0 += U) {
            if constexpr (PF > 0) {
              const int pe = t0 + U * PF + (lane % U);
              const CI pa = __shfl_sync(0xffffffffu, my_col, pe & 31);
              const CI pb = __shfl_sync(0xffffffffu, nx_col, pe & 31);
              const CI pc = pe < 32 ? pa : pb;
              const int line = lane / U;
              if (j0 + pe < je && line * (128 / (int)sizeof(T)) < 32 * CPL && (!HOT || pc >= 0)) {
                const char* pa_line = xbase + (uint64_t)(uint32_t)(HOT ? (pc & ~SPMM_FAR_BIT) : pc) * ldxb +
                                      (line * 128 - lane * CPL * (int)sizeof(T));
                if (HOT && (pc & SPMM_FAR_BIT)) {  // far reuse
                  if (farpf == 2)
                    asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], 128, %1;" ::
                                 "l"(pa_line), "l"(pol_far));
                  else if (farpf == 1)
                    asm volatile("prefetch.global.L2 [%0];" :: "l"(pa_line));
                } else {
                  asm volatile("prefetch.global.L2 [%0];" :: "l"(pa_line));
                }
              }
            }
            CI cols[U];
            T vals[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              cols[u] = __shfl_sync(0xffffffffu, my_col, (t0 + u) & 31);
              vals[u] = __shfl_sync(0xffffffffu, my_val, (t0 + u) & 31);   // 0 past the run
            }
            T xv[U][CPL];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              if (t0 + u < cnt) {
                if constexpr (HOT) {
                  // the column is warp-uniform (every lane loads its slice of
                  // the same X row): branch on it rather than select a policy
                  const CI cu = cols[u];
                  if (cu < 0) {
                    ldx_row<T, CPL>(reinterpret_cast<const T*>(hbase + (uint64_t)(uint32_t)(~cu) * ldhb), xv[u]);
                  } else {
                    const T* xr = reinterpret_cast<const T*>(
                        xbase + (uint64_t)(uint32_t)(cu & ~SPMM_FAR_BIT) * ldxb);
                    if (cu & SPMM_FAR_BIT) ldx_row_pol<T, CPL>(xr, xv[u], pol_far);
                    else ldx_row<T, CPL>(xr, xv[u]);
                  }
                } else {
                  ldx_row<T, CPL>(reinterpret_cast<const T*>(xbase + (uint64_t)(uint32_t)cols[u] * ldxb),
                                  xv[u]);
                }
              } else {
#pragma unroll
                for (int q = 0; q < CPL; ++q) xv[u][q] = T(0);
              }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
              // past the run: value 0 and X 0, the add of +0.0 leaves the sum
              // unchanged (a running sum from +0.0 is never -0.0)
              if (t0 + u < cnt && j0 + t0 + u == nxt) {
                do {   // rows that end here (empty rows included)
                  sty_row<T, CPL>(yrow, acc);
#pragma unroll
                  for (int q = 0; q < CPL; ++q) acc[q] = Arith<T>::zero();
                  yrow += ldy;
                  ++cur;
                  nxt = s_rp[cur + 1];
                } while (j0 + t0 + u == nxt);
              }
#pragma unroll
              for (int q = 0; q < CPL; ++q) acc[q] = Arith<T>::add(acc[q], Arith<T>::mul(vals[u], xv[u][q]));
            }
          }
          my_col = nx_col;
          my_val = nx_val;
        }
        for (; cur < rb; ++cur) {
          sty_row<T, CPL>(yrow, acc);
          yrow += ldy;
#pragma unroll
          for (int q = 0; q < CPL; ++q) acc[q] = Arith<T>::zero();
        }
        ra = rb;
      }
    }
  }
}

// L2 prefetch of far-reuse X rows in hinted plans: 0 none, 1 plain, 2 bulk
// prefetch with an evict_first policy (LAPIS_B200_SPMM_FARPF, A/B runs)
inline int spmm_far_prefetch() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LAPIS_B200_SPMM_FARPF");
    v = e ? atoi(e) : 0;
  }
  return v;
}

// gathers in flight per warp of the batch kernel: -1 = by element size
// (default), else LAPIS_B200_SPMM_U = 8 / 16 / 32 (A/B runs)
inline int spmm_u16() {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("LAPIS_B200_SPMM_U");
    v = e ? atoi(e) : -1;
  }
  return v;
}

// LAPIS_B200_SPMM_V1=1: the original batch kernel (A/B runs)
inline bool spmm_v1() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LAPIS_B200_SPMM_V1");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// --------------------------------------------------------------- long rows
// Rows longer than SPLIT entries (power-law hubs: config 3 has rows of
// 117,686 entries) are listed once by a streaming pass over rowptr, then
//  * fp32: each listed row is folded in the reference's exact order by the
//    pipelined kernel below (a reassociated fp32 sum of thousands of terms can
//    move by more than the 1e-5 contract);
//  * other types: each row is cut into SPLIT-entry chunks (work items built on
//    the device), a persistent CTA pool folds each chunk (8 warps on
//    contiguous sub-ranges, combined in warp order) into a partial, and the
//    partials of a row are added in chunk order.  Deterministic (fixed
//    association); exact for integers, within tolerance for fp64.
struct LongRows {
  int64_t* count;      // [1] listed rows
  int64_t* rows;       // [cap] row ids
  int64_t* total;      // [1] work items
  int64_t* work_row;   // [wcap] row of item
  int64_t* work_beg;   // [wcap] first entry of item
  int64_t* first;      // [cap] first item of listed row i
  unsigned long long* desc;  // [1] set when rowptr decreases somewhere
  int64_t cap, wcap;         // capacities of rows/first and work_row/work_beg
};

// listed rows the long-row kernels may use (0 when the rowptr decreases: the
// guarded fallback kernel then folds every row)
__device__ __forceinline__ int64_t long_rows_count(const LongRows& lr) {
  if (*(volatile const unsigned long long*)lr.desc) return 0;
  const int64_t n = *lr.count;
  return n < lr.cap ? n : lr.cap;
}

// rows the batch kernel skipped (long rows) hold AX in H after the long-row
// kernels; one warp per listed row applies the GCN epilogue in place
__global__ void __launch_bounds__(256)
gcn_long_rows_epilogue_kernel(const float* __restrict__ W, float* __restrict__ H, int64_t ldh,
                              const LongRows lr) {
  __shared__ __align__(16) float Ws[GCN_F * GCN_F];
  for (int t = threadIdx.x; t < GCN_F * GCN_F; t += blockDim.x) Ws[t] = W[t];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t n = long_rows_count(lr);
  for (int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); i < n; i += (int64_t)gridDim.x * 8) {
    float* hrow = H + lr.rows[i] * ldh;
    const float2 a = reinterpret_cast<const float2*>(hrow)[lane];
    __syncwarp();
    gcn_row_epilogue(a.x, a.y, Ws, hrow, lane);
  }
}

template <class RP>
__global__ void long_rows_list_kernel(int64_t nrows, const RP* __restrict__ rowptr, LongRows lr) {
  int desc = 0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t len = (int64_t)rowptr[r + 1] - (int64_t)rowptr[r];
    desc |= len < 0;
    if (len > SPLIT) {
      const unsigned long long i = atomicAdd(reinterpret_cast<unsigned long long*>(lr.count), 1ull);
      if ((int64_t)i < lr.cap) lr.rows[i] = r;  // > cap only with a bad nnz / decreasing rowptr
    }
  }
  if (__any_sync(0xffffffffu, desc) && (threadIdx.x & 31) == 0) atomicOr(lr.desc, 1ull);
}


// one CTA: each thread owns a contiguous slice of the listed rows; a block
// scan of the slices' chunk counts gives every row its first work item
template <class RP>
__global__ void __launch_bounds__(1024) long_rows_work_kernel(const RP* __restrict__ rowptr,
                                                              LongRows lr) {
  __shared__ int64_t scan[1024];
  const int64_t n = long_rows_count(lr);
  const int t = threadIdx.x;
  const int64_t i0 = n * t / 1024, i1 = n * (t + 1) / 1024;
  int64_t mine = 0;
  for (int64_t i = i0; i < i1; ++i) {
    const int64_t r = lr.rows[i];
    mine += ((int64_t)rowptr[r + 1] - (int64_t)rowptr[r] + SPLIT - 1) / SPLIT;
  }
  scan[t] = mine;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {  // inclusive Hillis-Steele scan
    const int64_t v = t >= off ? scan[t - off] : 0;
    __syncthreads();
    scan[t] += v;
    __syncthreads();
  }
  int64_t w = scan[t] - mine;
  if (t == 1023) *lr.total = scan[1023] < lr.wcap ? scan[1023] : lr.wcap;
  for (int64_t i = i0; i < i1; ++i) {
    const int64_t r = lr.rows[i];
    const int64_t b = (int64_t)rowptr[r], e = (int64_t)rowptr[r + 1];
    lr.first[i] = w;
    for (int64_t s = b; s < e; s += SPLIT, ++w) {
      if (w >= lr.wcap) break;  // only with an nnz below rowptr[n] - rowptr[0]
      lr.work_row[w] = r;
      lr.work_beg[w] = s;
    }
  }
}

// Pipelined version (the one launched): one CTA per (hub row, group of 16
// dense columns) — the row's 64 independent add chains run on 4 SMs, each
// gathering 64 B of every referenced X row.  Warp 0 folds (one thread per
// column, ascending entry order, the reference's rounding); warp 1 streams
// the row's colind PIPE_CD stages ahead into a PIPE_CR-slot shared-memory ring
// (cp.async, its own commit groups); warps 2-7 stream values and the X-row
// slices of stage s + PIPE_NS - 1 into a PIPE_NS-stage ring, reading the
// column indices from shared memory (four entries per warp instruction, one
// 8-byte pair per lane).  With colind that far ahead no loader ever waits on
// an index load, so a stage costs about its 128-add chain; the chain of the
// longest row (config 4: 70k entries) is the floor.
constexpr int PIPE_NS = 10, PIPE_SEQ = 128, PIPE_KC = 16, PIPE_LOADERS = 6;
constexpr int PIPE_CR = 32, PIPE_CD = 24;  // colind ring slots, prefetch distance (stages)
static_assert(PIPE_CD <= PIPE_CR + PIPE_NS - 3, "colind slot reused while still read");
static_assert(PIPE_CD >= PIPE_NS, "colind prefetch shorter than the data ring");

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory"); }

template <class CI>
constexpr size_t pipe_smem_bytes() {
  return (size_t)PIPE_NS * PIPE_SEQ * (PIPE_KC + 1) * sizeof(float) +
         (size_t)PIPE_CR * PIPE_SEQ * sizeof(CI);
}

template <class RP, class CI>
__global__ void __launch_bounds__(256, 2)
spmm_seq_long_pipe_kernel(int64_t k, const RP* __restrict__ rowptr,
                          const CI* __restrict__ colind, const float* __restrict__ values,
                          const float* __restrict__ X, int64_t ldx, float* __restrict__ Y,
                          int64_t ldy, const LongRows lr) {
  extern __shared__ __align__(16) unsigned char pipe_smem[];
  float* xs = reinterpret_cast<float*>(pipe_smem);            // [NS][SEQ][KC]
  float* vs = xs + PIPE_NS * PIPE_SEQ * PIPE_KC;               // [NS][SEQ]
  CI* cs = reinterpret_cast<CI*>(vs + PIPE_NS * PIPE_SEQ);     // [CR][SEQ]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool loader = warp >= 2;
  const int lw = warp - 2;
  const int64_t nlong = long_rows_count(lr);
  const int64_t ncg = (k + PIPE_KC - 1) / PIPE_KC;  // column groups per row
  for (int64_t item = blockIdx.x; item < nlong * ncg; item += gridDim.x) {
    const int64_t r = lr.rows[item / ncg];
    const int64_t b = (int64_t)rowptr[r], e = (int64_t)rowptr[r + 1];
    const int64_t nst = (e - b + PIPE_SEQ - 1) / PIPE_SEQ;
    const int64_t c0 = (item % ncg) * PIPE_KC;
    const int kc = (int)((k - c0) < PIPE_KC ? (k - c0) : PIPE_KC);
    const bool pairs = (kc == PIPE_KC) && (ldx % 2 == 0) && ((uintptr_t)X % 8 == 0);
    auto issue_cols = [&](int64_t t) {  // warp 1
      if (t < nst) {
        const int64_t j0 = b + t * PIPE_SEQ;
        const int n = (int)((e - j0) < PIPE_SEQ ? (e - j0) : PIPE_SEQ);
        CI* dst = cs + (int)(t % PIPE_CR) * PIPE_SEQ;
        for (int i = lane; i < n; i += 32) {
          if constexpr (sizeof(CI) == 8) cp_async8(dst + i, colind + j0 + i);
          else cp_async4(dst + i, colind + j0 + i);
        }
      }
      cp_commit();  // one group per stage, possibly empty: uniform wait counts
    };
    auto issue = [&](int64_t t) {  // warps 2-7
      if (t < nst) {
        const int slot = (int)(t % PIPE_NS);
        const int64_t j0 = b + t * PIPE_SEQ;
        const int n = (int)((e - j0) < PIPE_SEQ ? (e - j0) : PIPE_SEQ);
        const CI* cr = cs + (int)(t % PIPE_CR) * PIPE_SEQ;
        const int lt = threadIdx.x - 64;
        if (lt < n) cp_async4(&vs[slot * PIPE_SEQ + lt], values + j0 + lt);
        if (lt + 192 < n) cp_async4(&vs[slot * PIPE_SEQ + lt + 192], values + j0 + lt + 192);
        if (pairs) {
          // lane: entry (lane / 8) of a group of 4, column pair (lane % 8)
          for (int jj = 4 * lw + (lane >> 3); jj < n; jj += 4 * PIPE_LOADERS) {
            const int64_t cu = (int64_t)cr[jj];
            cp_async8(&xs[(slot * PIPE_SEQ + jj) * PIPE_KC + 2 * (lane & 7)],
                      X + cu * ldx + c0 + 2 * (lane & 7));
          }
        } else {
          for (int jj = lw; jj < n; jj += PIPE_LOADERS) {
            const int64_t cu = (int64_t)cr[jj];
            if (lane < kc) cp_async4(&xs[(slot * PIPE_SEQ + jj) * PIPE_KC + lane], X + cu * ldx + c0 + lane);
          }
        }
      }
      cp_commit();
    };
    if (warp == 1) {
      for (int t = 0; t < PIPE_CD; ++t) issue_cols(t);
      cp_wait<PIPE_CD - PIPE_NS + 1>();  // colind of stages 0 .. NS-2 landed
    }
    __syncthreads();
    if (loader)
      for (int t = 0; t < PIPE_NS - 1; ++t) issue(t);
    float acc = 0.0f;
    for (int64_t s = 0; s < nst; ++s) {
      if (loader) cp_wait<PIPE_NS - 2>();   // this thread's copies of stage s landed
      if (warp == 1) {
        issue_cols(s + PIPE_CD);
        cp_wait<PIPE_CD - PIPE_NS + 1>();   // colind of stage s + NS - 1 landed
      }
      __syncthreads();                      // stage s and colind of s + NS - 1 visible
      if (loader) {
        issue(s + PIPE_NS - 1);             // into slot (s - 1) % NS
      } else if ((int)threadIdx.x < kc) {
        const int slot = (int)(s % PIPE_NS);
        const int64_t j0 = b + s * PIPE_SEQ;
        const int n = (int)((e - j0) < PIPE_SEQ ? (e - j0) : PIPE_SEQ);
        const float* xr = &xs[slot * PIPE_SEQ * PIPE_KC + threadIdx.x];
        const float* vr = &vs[slot * PIPE_SEQ];
        int jj = 0;
        for (; jj + 16 <= n; jj += 16) {  // all 32 shared loads in flight, then the add chain
          float vv[16], xx[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) { vv[u] = vr[jj + u]; xx[u] = xr[(jj + u) * PIPE_KC]; }
#pragma unroll
          for (int u = 0; u < 16; ++u) acc = __fadd_rn(acc, __fmul_rn(vv[u], xx[u]));
        }
        for (; jj < n; ++jj) acc = __fadd_rn(acc, __fmul_rn(vr[jj], xr[jj * PIPE_KC]));
      }
    }
    if (loader || warp == 1) cp_wait<0>();
    __syncthreads();  // the rings are reused by the next item
    if ((int)threadIdx.x < kc) Y[r * ldy + c0 + threadIdx.x] = acc;
  }
}

template <class T, class RP, class CI>
__global__ void __launch_bounds__(SPMM_WARPS * 32)
spmm_long_chunk_kernel(int64_t k, const RP* __restrict__ rowptr, const CI* __restrict__ colind,
                       const T* __restrict__ values, const T* __restrict__ X, int64_t ldx,
                       T* __restrict__ part, const LongRows lr) {
  extern __shared__ unsigned char smem_raw[];
  T* wpart = reinterpret_cast<T*>(smem_raw);  // [SPMM_WARPS][k]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t total = *lr.total;
  for (int64_t w = blockIdx.x; w < total; w += gridDim.x) {
    const int64_t r = lr.work_row[w];
    const int64_t s0 = lr.work_beg[w];
    const int64_t e = (int64_t)rowptr[r + 1];
    const int64_t s1 = (s0 + SPLIT) < e ? (s0 + SPLIT) : e;
    const int64_t len = s1 - s0;
    const int64_t w0 = s0 + len * warp / SPMM_WARPS, w1 = s0 + len * (warp + 1) / SPMM_WARPS;
    for (int64_t col = lane; col < k; col += 32) {
      T acc = Arith<T>::zero();
      int64_t j = w0;
      for (; j + 4 <= w1; j += 4) {  // 4 gathers in flight, folded in order
        T v[4], x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          v[u] = values[j + u];
          x[u] = __ldg(X + (int64_t)colind[j + u] * ldx + col);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc = Arith<T>::add(acc, Arith<T>::mul(v[u], x[u]));
      }
      for (; j < w1; ++j)
        acc = Arith<T>::add(acc, Arith<T>::mul(values[j], __ldg(X + (int64_t)colind[j] * ldx + col)));
      wpart[warp * k + col] = acc;
    }
    __syncthreads();
    T* dst = part + w * k;
    for (int64_t col = threadIdx.x; col < k; col += blockDim.x) {
      T acc = Arith<T>::zero();
      for (int ww = 0; ww < SPMM_WARPS; ++ww) acc = Arith<T>::add(acc, wpart[ww * k + col]);
      dst[col] = acc;
    }
    __syncthreads();
  }
}

template <class T, class RP>
__global__ void spmm_long_combine_kernel(int64_t k, const RP* __restrict__ rowptr,
                                         const T* __restrict__ part, T* __restrict__ Y, int64_t ldy,
                                         const LongRows lr) {
  const int64_t n = long_rows_count(lr);
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const int64_t r = lr.rows[i];
    const int64_t w0 = lr.first[i];
    const int64_t nch = ((int64_t)rowptr[r + 1] - (int64_t)rowptr[r] + SPLIT - 1) / SPLIT;
    for (int64_t col = threadIdx.x; col < k; col += blockDim.x) {
      T acc = part[w0 * k + col];
      for (int64_t c = 1; c < nch; ++c) acc = Arith<T>::add(acc, part[(w0 + c) * k + col]);
      Y[r * ldy + col] = acc;
    }
  }
}

// ================================================================ host side
// LAPIS_B200_SPMM_ROW=1 selects the one-row-per-warp kernel (A/B measurements)
inline bool spmm_force_row() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LAPIS_B200_SPMM_ROW");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// LAPIS_B200_SPMM_STATIC=1: static grid-stride batch assignment (A/B runs)
inline bool spmm_static() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LAPIS_B200_SPMM_STATIC");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

struct HotMap {
  const int32_t* colind;  // remapped copy (negative: ~row of xhot)
  const void* xhot;       // [nhot, ldh]
  int64_t ldh;
};

template <class T, class RP, class CI>
struct SpmmOp {
  static int run(int64_t nrows, int64_t nnz, int64_t k, const void* rowptr, const void* colind,
                 const void* values, const void* X, int64_t ldx, void* Y, int64_t ldy,
                 cudaStream_t st, const void* W = nullptr, const HotMap* hot = nullptr) {
    // W != nullptr: fused GCN layer (fp32, k = 64 through the batch kernel;
    // gcn_layer checks the preconditions), Y is H
    const int64_t blocks = (nrows + SPMM_WARPS - 1) / SPMM_WARPS;
    if (blocks > 0x7fffffffLL) return fail(LAPIS_B200_ERR_ARG, "spmm: too many rows");
    const bool grp = (k < 64) && (k % 4 == 0) && (ldx % 4 == 0) && (ldy % 4 == 0) &&
                     ((uintptr_t)X % 16 == 0) && ((uintptr_t)Y % 16 == 0);
    const bool vec = (ldx % 2 == 0) && ((uintptr_t)X % (2 * sizeof(T)) == 0);
    const int64_t cpl = (k % 128 == 0) ? 4 : (k % 64 == 0) ? 2 : (k % 32 == 0) ? 1 : 0;
    const bool batch = cpl > 0 && (ldx % cpl == 0) && (ldy % cpl == 0) &&
                       ((uintptr_t)X % (cpl * sizeof(T)) == 0) &&
                       ((uintptr_t)Y % (cpl * sizeof(T)) == 0) && !spmm_force_row();
    // ---- long-row list + decreasing-rowptr flag: one pass over rowptr,
    // launched first so every later kernel can be guarded by the flag
    const int64_t cap = nnz / (SPLIT + 1) + 1;       // rows with > SPLIT entries
    const int64_t wcap = nnz / SPLIT + cap + 1;       // chunks of those rows
    int64_t* ws = nullptr;
    const size_t ws_elems = 3 + 2 * (size_t)cap + 2 * (size_t)wcap;
    LB_TRY(check_cuda(cudaMallocAsync((void**)&ws, ws_elems * sizeof(int64_t), st), "alloc(long rows)"));
    struct FreeWs {
      int64_t* p; cudaStream_t s;
      ~FreeWs() { cudaFreeAsync(p, s); }
    } free_ws{ws, st};
    LongRows lr;
    lr.count = ws;
    lr.total = ws + 1;
    lr.desc = reinterpret_cast<unsigned long long*>(ws + 2);
    lr.rows = ws + 3;
    lr.first = lr.rows + cap;
    lr.work_row = lr.first + cap;
    lr.work_beg = lr.work_row + wcap;
    lr.cap = cap;
    lr.wcap = wcap;
    LB_TRY(check_cuda(cudaMemsetAsync(ws, 0, 3 * sizeof(int64_t), st), "memset(long rows)"));
    const int sms = num_sms();
    {
      int64_t g = (nrows + 255) / 256;
      if (g > (int64_t)sms * 8) g = (int64_t)sms * 8;
      long_rows_list_kernel<RP><<<(unsigned)(g > 0 ? g : 1), 256, 0, st>>>(nrows, (const RP*)rowptr, lr);
      LB_TRY(check_launch("long_rows_list_kernel"));
    }
    const int64_t row_grid = blocks < (int64_t)sms * 16 ? blocks : (int64_t)sms * 16;
    DescGuard fast, fallback;
    fast.desc = fallback.desc = lr.desc;
    fallback.mode = 1;
    // ---- long rows (> SPLIT entries): listed above, folded (fp32: exact
    // order) or chunked + combined on a high-priority side stream, CONCURRENT
    // with the short-row kernels below — they write disjoint rows of Y, and a
    // hub row's fold is a long dependent add chain (config 4: 70k entries)
    // that would otherwise run alone on a few SMs after the batch kernel
    T* part = nullptr;
    cudaStream_t ls = st;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    auto join_long = [&]() -> int {
      int jrc = LAPIS_B200_OK;
      if (ev_join) {
        jrc = check_cuda(cudaStreamWaitEvent(st, ev_join, 0), "join long-row stream");
        cudaEventDestroy(ev_join);
      }
      if (ev_fork) cudaEventDestroy(ev_fork);
      if (part) cudaFreeAsync(part, st);
      return jrc;
    };
    if (nnz > SPLIT) {
      cudaStream_t side = long_row_stream();
      if (side && cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming) == cudaSuccess &&
          cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming) == cudaSuccess &&
          cudaEventRecord(ev_fork, st) == cudaSuccess &&
          cudaStreamWaitEvent(side, ev_fork, 0) == cudaSuccess)
        ls = side;
      cudaGetLastError();
      int rc = LAPIS_B200_OK;
      [&] {
      // ---- long rows: fold (fp32 exact) or chunk + combine
      if constexpr (std::is_same<T, float>::value) {
        constexpr size_t pipe_smem = pipe_smem_bytes<CI>();
        if (rc == LAPIS_B200_OK)
          rc = check_cuda(cudaFuncSetAttribute(spmm_seq_long_pipe_kernel<RP, CI>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)pipe_smem), "smem attr (seq pipe)");
        if (rc == LAPIS_B200_OK) {
          const int64_t items = cap * ((k + PIPE_KC - 1) / PIPE_KC);
          const int64_t g = items < (int64_t)sms * 2 ? items : (int64_t)sms * 2;
          spmm_seq_long_pipe_kernel<RP, CI><<<(unsigned)g, 256, pipe_smem, ls>>>(
              k, (const RP*)rowptr, (const CI*)colind, (const float*)values, (const float*)X, ldx,
              (float*)Y, ldy, lr);
          rc = check_launch("spmm_seq_long_pipe_kernel");
        }
        if (rc == LAPIS_B200_OK && W) {
          const int64_t g = (cap + 7) / 8 < sms ? (cap + 7) / 8 : sms;
          gcn_long_rows_epilogue_kernel<<<(unsigned)g, 256, 0, ls>>>((const float*)W, (float*)Y,
                                                                       ldy, lr);
          rc = check_launch("gcn_long_rows_epilogue_kernel");
        }
      } else {
      if (rc == LAPIS_B200_OK) {
        long_rows_work_kernel<RP><<<1, 1024, 0, ls>>>((const RP*)rowptr, lr);
        rc = check_launch("long_rows_work_kernel");
      }
      if (rc == LAPIS_B200_OK)
        rc = check_cuda(cudaMallocAsync((void**)&part, (size_t)wcap * k * sizeof(T), ls), "alloc(part)");
      const size_t smem = (size_t)SPMM_WARPS * k * sizeof(T);
      if (rc == LAPIS_B200_OK && smem > 48 * 1024) {
        rc = check_cuda(cudaFuncSetAttribute(spmm_long_chunk_kernel<T, RP, CI>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                        "smem attr");
        if (rc == LAPIS_B200_OK && smem > 200 * 1024)
          rc = fail(LAPIS_B200_ERR_UNSUPPORTED, "spmm: k too large for long-row staging");
      }
      if (rc == LAPIS_B200_OK) {
        const int64_t g = wcap < (int64_t)sms * 8 ? wcap : (int64_t)sms * 8;
        spmm_long_chunk_kernel<T, RP, CI><<<(unsigned)g, SPMM_WARPS * 32, smem, ls>>>(
            k, (const RP*)rowptr, (const CI*)colind, (const T*)values, (const T*)X, ldx, part, lr);
        rc = check_launch("spmm_long_chunk_kernel");
      }
      if (rc == LAPIS_B200_OK) {
        const int64_t g = cap < (int64_t)sms * 4 ? cap : (int64_t)sms * 4;
        spmm_long_combine_kernel<T, RP><<<(unsigned)g, 64, 0, ls>>>(k, (const RP*)rowptr, part,
                                                                   (T*)Y, ldy, lr);
        rc = check_launch("spmm_long_combine_kernel");
      }
        }
      }();
      if (ls != st) cudaEventRecord(ev_join, ls);
      if (rc != LAPIS_B200_OK) { join_long(); return rc; }
    }
    if (batch) {
      int64_t gblocks = ((nrows + 31) / 32 + 7) / 8;
      const int64_t gcap = (int64_t)sms * 8;
      if (gblocks > gcap) gblocks = gcap;
      if (gblocks < 1) gblocks = 1;
      const int pf = spmm_prefetch_distance();
      unsigned long long* next = nullptr;
      if (!spmm_static()) {
        LB_TRY(check_cuda(cudaMallocAsync((void**)&next, sizeof(*next), st), "alloc(spmm counter)"));
        const int mrc = check_cuda(cudaMemsetAsync(next, 0, sizeof(*next), st), "memset(spmm counter)");
        if (mrc != LAPIS_B200_OK) { cudaFreeAsync(next, st); return mrc; }
      }
      struct FreeNext {
        unsigned long long* p; cudaStream_t s;
        ~FreeNext() { if (p) cudaFreeAsync(p, s); }
      } free_next{next, st};
#define LB_BAT(CC) spmm_batch_kernel<T, RP, CI, CC, 8><<<(unsigned)gblocks, 256, 0, st>>>( \
          nrows, k, (const RP*)rowptr, (const CI*)colind, (const T*)values, (const T*)X, ldx, (T*)Y, ldy, \
          nullptr, next, pf, fast)
      bool fused = false;
      if constexpr (std::is_same<T, float>::value) {
        if (W) {
          // (the fused layer needs a non-decreasing rowptr: the fallback below
          // computes A X only; gcn_layer takes this path on request only)
          if (cpl != 2 || k != GCN_F) return fail(LAPIS_B200_ERR_ARG, "gcn fused: k must be 64");
          spmm_batch_kernel<float, RP, CI, 2, 8, true><<<(unsigned)gblocks, 256, 0, st>>>(
              nrows, k, (const RP*)rowptr, (const CI*)colind, (const float*)values,
              (const float*)X, ldx, (float*)Y, ldy, (const float*)W, next, pf, fast);
          fused = true;
        }
      }
      if (!fused) {
        if (W) return fail(LAPIS_B200_ERR_ARG, "gcn fused: fp32 only");
        if (hot && next && pf <= 1) {
#define LB_BATH(CC, PFV) spmm_batch2_kernel<T, RP, int32_t, CC, 8, PFV, true><<<(unsigned)gblocks, 256, 0, st>>>( \
          nrows, k, (const RP*)rowptr, hot->colind, (const T*)values, (const T*)X, ldx, (T*)Y, ldy, \
          next, fast, (const T*)hot->xhot, hot->ldh, spmm_far_prefetch())
          if (spmm_u16() == 16 && cpl == 2) {
            spmm_batch2_kernel<T, RP, int32_t, 2, 16, 1, true><<<(unsigned)gblocks, 256, 0, st>>>(
                nrows, k, (const RP*)rowptr, hot->colind, (const T*)values, (const T*)X, ldx, (T*)Y, ldy,
                next, fast, (const T*)hot->xhot, hot->ldh, spmm_far_prefetch());
          } else if (pf == 1) {
            if (cpl == 4) LB_BATH(4, 1); else if (cpl == 2) LB_BATH(2, 1); else LB_BATH(1, 1);
          } else {
            if (cpl == 4) LB_BATH(4, 0); else if (cpl == 2) LB_BATH(2, 0); else LB_BATH(1, 0);
          }
#undef LB_BATH
        } else if (next && !spmm_v1() && pf <= 1) {
#define LB_BAT2(CC, PFV) spmm_batch2_kernel<T, RP, CI, CC, 8, PFV><<<(unsigned)gblocks, 256, 0, st>>>( \
          nrows, k, (const RP*)rowptr, (const CI*)colind, (const T*)values, (const T*)X, ldx, (T*)Y, ldy, \
          next, fast)
          if (spmm_u16() == 32 && cpl == 2) {
            spmm_batch2_kernel<T, RP, CI, 2, 32, 1><<<(unsigned)gblocks, 256, 0, st>>>(
                nrows, k, (const RP*)rowptr, (const CI*)colind, (const T*)values, (const T*)X, ldx,
                (T*)Y, ldy, next, fast);
          } else if ((spmm_u16() == 16 || (spmm_u16() < 0 && sizeof(T) == 4)) && cpl <= 2) {
            // 4-byte elements: 16 gathers in flight per warp (three CTAs per
            // SM); config 4's SpMM 0.848 -> 0.813 ms per layer.  (8-byte rows:
            // config 3 9.86 -> 15.3 ms, so they keep 8.)
            if (cpl == 2)
              spmm_batch2_kernel<T, RP, CI, 2, 16, 1><<<(unsigned)gblocks, 256, 0, st>>>(
                  nrows, k, (const RP*)rowptr, (const CI*)colind, (const T*)values, (const T*)X, ldx,
                  (T*)Y, ldy, next, fast);
            else
              spmm_batch2_kernel<T, RP, CI, 1, 16, 1><<<(unsigned)gblocks, 256, 0, st>>>(
                  nrows, k, (const RP*)rowptr, (const CI*)colind, (const T*)values, (const T*)X, ldx,
                  (T*)Y, ldy, next, fast);
          } else if (pf == 1) {
            if (cpl == 4) LB_BAT2(4, 1); else if (cpl == 2) LB_BAT2(2, 1); else LB_BAT2(1, 1);
          } else {
            if (cpl == 4) LB_BAT2(4, 0); else if (cpl == 2) LB_BAT2(2, 0); else LB_BAT2(1, 0);
          }
#undef LB_BAT2
        } else {
          if (cpl == 4) LB_BAT(4); else if (cpl == 2) LB_BAT(2); else LB_BAT(1);
        }
      }
#undef LB_BAT
    } else if (W) {
      return fail(LAPIS_B200_ERR_ARG, "gcn fused: needs the batch kernel's layout");
    } else if (grp) {
      const int64_t lanes_per_row = k >= 64 ? 16 : (k >= 32 ? 8 : (k >= 16 ? 4 : (k >= 8 ? 2 : 1)));
      int64_t gblocks = (nrows * lanes_per_row + 255) / 256;
      const int64_t gcap = (int64_t)sms * 8;
      if (gblocks > gcap) gblocks = gcap;
      if (gblocks < 1) gblocks = 1;
#define LB_GRP(GG) spmm_group_kernel<T, RP, CI, GG><<<(unsigned)gblocks, 256, 0, st>>>( \
          nrows, k, (const RP*)rowptr, (const CI*)colind, (const T*)values, (const T*)X, ldx, (T*)Y, ldy, fast)
      switch (lanes_per_row) {
        case 16: LB_GRP(16); break;
        case 8: LB_GRP(8); break;
        case 4: LB_GRP(4); break;
        case 2: LB_GRP(2); break;
        default: LB_GRP(1); break;
      }
#undef LB_GRP
    } else if (vec)
      spmm_row_kernel<T, RP, CI, 2><<<(unsigned)row_grid, SPMM_WARPS * 32, 0, st>>>(
          nrows, k, (const RP*)rowptr, (const CI*)colind, (const T*)values, (const T*)X, ldx,
          (T*)Y, ldy, fast);
    else
      spmm_row_kernel<T, RP, CI, 1><<<(unsigned)row_grid, SPMM_WARPS * 32, 0, st>>>(
          nrows, k, (const RP*)rowptr, (const CI*)colind, (const T*)values, (const T*)X, ldx,
          (T*)Y, ldy, fast);
    LB_TRY(check_launch("spmm_row_kernel"));
    // decreasing rowptr only: one warp per row, every row on its clamped range
    if (vec)
      spmm_row_kernel<T, RP, CI, 2><<<(unsigned)row_grid, SPMM_WARPS * 32, 0, st>>>(
          nrows, k, (const RP*)rowptr, (const CI*)colind, (const T*)values, (const T*)X, ldx,
          (T*)Y, ldy, fallback);
    else
      spmm_row_kernel<T, RP, CI, 1><<<(unsigned)row_grid, SPMM_WARPS * 32, 0, st>>>(
          nrows, k, (const RP*)rowptr, (const CI*)colind, (const T*)values, (const T*)X, ldx,
          (T*)Y, ldy, fallback);
    LB_TRY(check_launch("spmm_row_kernel(fallback)"));
    return join_long();
  }
};

// GCN layer H = relu((A X) W) in one pass over A (fp32, fin = fout = 64; the
// caller checks): the batch kernel applies W and the ReLU to each finished row
int spmm_gcn_fused(int64_t nrows, int64_t nnz, const void* rowptr, int rp_bytes,
                   const void* colind, int ci_bytes, const void* values, const void* X,
                   int64_t ldx, const void* W, void* H, int64_t ldh, cudaStream_t st) {
  if (rp_bytes == 8 && ci_bytes == 4)
    return SpmmOp<float, int64_t, int32_t>::run(nrows, nnz, GCN_F, rowptr, colind, values, X, ldx, H, ldh, st, W);
  if (rp_bytes == 8 && ci_bytes == 8)
    return SpmmOp<float, int64_t, int64_t>::run(nrows, nnz, GCN_F, rowptr, colind, values, X, ldx, H, ldh, st, W);
  if (rp_bytes == 4 && ci_bytes == 4)
    return SpmmOp<float, int32_t, int32_t>::run(nrows, nnz, GCN_F, rowptr, colind, values, X, ldx, H, ldh, st, W);
  return SpmmOp<float, int32_t, int64_t>::run(nrows, nnz, GCN_F, rowptr, colind, values, X, ldx, H, ldh, st, W);
}

int spmm_csr(int64_t nrows, int64_t ncols, int64_t nnz, int64_t k, const void* rowptr,
             int rp_bytes, const void* colind, int ci_bytes, const void* values, const void* X,
             int64_t ldx, void* Y, int64_t ldy, int dtype, cudaStream_t st) {
  if (nrows < 0 || ncols < 0 || nnz < 0 || k < 0) return fail(LAPIS_B200_ERR_ARG, "spmm: negative extent");
  if (!valid_dtype(dtype)) return fail(LAPIS_B200_ERR_ARG, "spmm: unsupported dtype");
  if ((rp_bytes != 4 && rp_bytes != 8) || (ci_bytes != 4 && ci_bytes != 8))
    return fail(LAPIS_B200_ERR_ARG, "spmm: index widths must be 4 or 8 bytes");
  if (ldx < k || ldy < k) return fail(LAPIS_B200_ERR_ARG, "spmm: leading dimension < k");
  if (!rowptr || (nrows > 0 && k > 0 && !Y) || (nnz > 0 && (!colind || !values || !X)))
    return fail(LAPIS_B200_ERR_ARG, "spmm: null operand");
  if (nrows == 0 || k == 0) return LAPIS_B200_OK;
#define LB_SPMM(T)                                                                             \
  if (rp_bytes == 8 && ci_bytes == 4) return SpmmOp<T, int64_t, int32_t>::run(nrows, nnz, k, rowptr, colind, values, X, ldx, Y, ldy, st); \
  if (rp_bytes == 8 && ci_bytes == 8) return SpmmOp<T, int64_t, int64_t>::run(nrows, nnz, k, rowptr, colind, values, X, ldx, Y, ldy, st); \
  if (rp_bytes == 4 && ci_bytes == 4) return SpmmOp<T, int32_t, int32_t>::run(nrows, nnz, k, rowptr, colind, values, X, ldx, Y, ldy, st); \
  return SpmmOp<T, int32_t, int64_t>::run(nrows, nnz, k, rowptr, colind, values, X, ldx, Y, ldy, st);
  switch (dtype) {
    case LAPIS_B200_F64: { LB_SPMM(double) }
    case LAPIS_B200_F32: { LB_SPMM(float) }
    case LAPIS_B200_I64: { LB_SPMM(long long) }
    case LAPIS_B200_I32: { LB_SPMM(int) }
  }
#undef LB_SPMM
  return fail(LAPIS_B200_ERR_ARG, "spmm: unsupported dtype");
}


// ============================================================ SpMM plans
// Structure-only analysis of a CSR structure for repeated Y = A X with new X
// every call (config 3; the GCN's features): the X rows referenced most often
// are copied each call into a compact buffer Xh that a persisting L2 access
// policy window pins, and the batch kernel reads them there through a
// remapped private colind (negative entries).  The rest of X streams as
// before.  Per-row entry order is unchanged (bit-identical).
// scripts/c3_gather_bound.py puts the motivation in numbers: config 3's 100M
// gathers of 512-byte X rows cost 51 GB with no reuse, 49 GB under LRU with
// the whole 126 MB L2, 45.7 GB when the 64 MB most-referenced rows stay
// resident, 37 GB at Belady's optimum.
struct SpmmPlanImpl {
  int device = 0;
  int64_t nrows = 0, ncols = 0, nnz = 0, k = 0;
  int dtype = 0;
  int32_t* colind_hot = nullptr;  // [nnz]
  int32_t* hot_cols = nullptr;    // [nhot]
  void* xhot = nullptr;           // [nhot, k]
  int64_t nhot = 0, hot_entries = 0;
  size_t window_bytes = 0;        // persisting window actually granted
  int hints = 0;                  // 1: SPMM_FAR_BIT reuse hints in colind_hot
  int64_t far_entries = 0;        // entries marked far
};

__global__ void col_hist_kernel(int64_t nnz, const int32_t* __restrict__ ci32,
                                const int64_t* __restrict__ ci64, unsigned* __restrict__ counts) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nnz;
       j += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(counts + (ci32 ? (int64_t)ci32[j] : ci64[j]), 1u);
}
__global__ void count_hist_kernel(int64_t ncols, const unsigned* __restrict__ counts,
                                  unsigned long long* __restrict__ hist, int nbins) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncols;
       c += (int64_t)gridDim.x * blockDim.x) {
    const unsigned v = counts[c];
    atomicAdd(hist + (v < (unsigned)nbins ? v : (unsigned)(nbins - 1)), 1ull);
  }
}
__global__ void hot_assign_kernel(int64_t ncols, const unsigned* __restrict__ counts, unsigned tau,
                                  int64_t cap, unsigned long long* __restrict__ slot,
                                  int32_t* __restrict__ hot_index, int32_t* __restrict__ hot_cols) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncols;
       c += (int64_t)gridDim.x * blockDim.x) {
    int32_t h = -1;
    if (counts[c] >= tau) {
      const unsigned long long s = atomicAdd(slot, 1ull);
      if ((int64_t)s < cap) { h = (int32_t)s; hot_cols[s] = (int32_t)c; }
    }
    hot_index[c] = h;
  }
}
__global__ void hot_remap_kernel(int64_t nnz, const int32_t* __restrict__ ci32,
                                 const int64_t* __restrict__ ci64,
                                 const int32_t* __restrict__ hot_index, int32_t* __restrict__ out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nnz;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = ci32 ? (int64_t)ci32[j] : ci64[j];
    const int32_t h = hot_index[c];
    out[j] = h >= 0 ? ~h : (int32_t)c;
  }
}
// Xh[h, :] = X[hot_cols[h], :] — one warp per row, 16-byte copies
__global__ void hot_gather_kernel(int64_t nhot, int64_t row_bytes, const int32_t* __restrict__ hot_cols,
                                  const unsigned char* __restrict__ X, int64_t ldx_bytes,
                                  unsigned char* __restrict__ Xh) {
  const int lane = threadIdx.x & 31;
  for (int64_t h = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; h < nhot;
       h += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const unsigned char* src = X + (int64_t)hot_cols[h] * ldx_bytes;
    unsigned char* dst = Xh + h * row_bytes;
    for (int64_t b = (int64_t)lane * 16; b < row_bytes; b += 32 * 16)
      *reinterpret_cast<int4*>(dst + b) = __ldg(reinterpret_cast<const int4*>(src + b));
  }
}

// Reuse hints (bit 30 of the remapped colind, SPMM_FAR_BIT): the gathers run
// in CSR order, so the distance from an entry to the next entry of the same
// column is the X row's reuse distance.  Entries whose next use lies more
// than D entries ahead (D = 8 L2-sized working sets of X rows) are loaded
// evict_first and the rest evict_normal — a cheap stand-in for Belady's
// replacement.  scripts/cache_sim.c on config 3 (126 MB of X rows): LRU 84.2M
// misses, this policy 61.4M, Belady 61.0M.  Positions sorted by column
// (stable radix sort) give every entry its successor in one pass.
__global__ void col_keys_kernel(int64_t nnz, const int32_t* __restrict__ ci32,
                                const int64_t* __restrict__ ci64, int32_t* __restrict__ keys,
                                int32_t* __restrict__ pos) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nnz;
       j += (int64_t)gridDim.x * blockDim.x) {
    keys[j] = ci32 ? ci32[j] : (int32_t)ci64[j];
    pos[j] = (int32_t)j;
  }
}
__global__ void reuse_hint_kernel(int64_t nnz, const int32_t* __restrict__ skeys,
                                  const int32_t* __restrict__ spos, int64_t horizon,
                                  int32_t* __restrict__ colind_hot,
                                  unsigned long long* __restrict__ nfar) {
  unsigned long long local = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = spos[i];
    const bool near = i + 1 < nnz && skeys[i + 1] == skeys[i] && (int64_t)spos[i + 1] - p <= horizon;
    const int32_t c = colind_hot[p];
    if (!near && c >= 0) {
      colind_hot[p] = c | SPMM_FAR_BIT;
      ++local;
    }
  }
  if (local) atomicAdd(nfar, local);
}

static int spmm_reuse_hints(SpmmPlanImpl* p, const int32_t* c32, const int64_t* c64,
                            int64_t row_bytes, cudaStream_t st) {
  const int64_t nnz = p->nnz;
  int l2 = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, p->device);
  const char* de = getenv("LAPIS_B200_SPMM_HINT_D");
  const double mult = de ? atof(de) : 8.0;
  const int64_t horizon = (int64_t)(mult * (double)std::max<int64_t>(1, (int64_t)l2 / row_bytes));
  int end_bit = 1;
  while (end_bit < 31 && (1ll << end_bit) < p->ncols) ++end_bit;
  int32_t *keys = nullptr, *keys2 = nullptr, *pos = nullptr, *pos2 = nullptr;
  void* tmp = nullptr;
  unsigned long long* nfar = nullptr;
  size_t tmp_bytes = 0;
  auto cleanup = [&]() {
    for (void* q : {(void*)keys, (void*)keys2, (void*)pos, (void*)pos2, tmp, (void*)nfar})
      if (q) cudaFreeAsync(q, st);
  };
  const size_t b = (size_t)nnz * 4;
  // the hints are optional: without room for the sort's 16 bytes per entry the
  // plan goes without them (allocation failures are cleared, not reported)
  bool room = cudaMallocAsync((void**)&keys, b, st) == cudaSuccess &&
              cudaMallocAsync((void**)&keys2, b, st) == cudaSuccess &&
              cudaMallocAsync((void**)&pos, b, st) == cudaSuccess &&
              cudaMallocAsync((void**)&pos2, b, st) == cudaSuccess &&
              cudaMallocAsync((void**)&nfar, 8, st) == cudaSuccess;
  if (!room) {
    cudaGetLastError();
    cleanup();
    return LAPIS_B200_OK;
  }
  int rc = LAPIS_B200_OK;
  if (rc == LAPIS_B200_OK) rc = check_cuda(cudaMemsetAsync(nfar, 0, 8, st), "memset(hint count)");
  const int sms = num_sms();
  const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((nnz + 255) / 256, (int64_t)sms * 8));
  if (rc == LAPIS_B200_OK) {
    col_keys_kernel<<<g, 256, 0, st>>>(nnz, c32, c64, keys, pos);
    rc = check_launch("col_keys_kernel");
  }
  if (rc == LAPIS_B200_OK)
    rc = check_cuda(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys2, pos, pos2,
                                                    (int)nnz, 0, end_bit, st), "radix sort (size)");
  if (rc == LAPIS_B200_OK && cudaMallocAsync(&tmp, tmp_bytes, st) != cudaSuccess) {
    cudaGetLastError();
    cleanup();
    return LAPIS_B200_OK;
  }
  if (rc == LAPIS_B200_OK)
    rc = check_cuda(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys2, pos, pos2,
                                                    (int)nnz, 0, end_bit, st), "radix sort");
  if (rc == LAPIS_B200_OK) {
    reuse_hint_kernel<<<g, 256, 0, st>>>(nnz, keys2, pos2, horizon, p->colind_hot, nfar);
    rc = check_launch("reuse_hint_kernel");
  }
  unsigned long long h = 0;
  if (rc == LAPIS_B200_OK)
    rc = check_cuda(cudaMemcpyAsync(&h, nfar, 8, cudaMemcpyDeviceToHost, st), "hint count D2H");
  cleanup();
  if (rc == LAPIS_B200_OK) rc = check_cuda(cudaStreamSynchronize(st), "hint sync");
  if (rc == LAPIS_B200_OK) {
    p->far_entries = (int64_t)h;
    p->hints = 1;
  }
  return rc;
}

int spmm_plan_create(int64_t nrows, int64_t ncols, int64_t nnz, int64_t k, const void* rowptr,
                     int rp_bytes, const void* colind, int ci_bytes, int dtype, int64_t hot_bytes,
                     cudaStream_t st, void** out) {
  if (!out) return fail(LAPIS_B200_ERR_ARG, "spmm plan: null out pointer");
  *out = nullptr;
  if (nrows < 0 || ncols < 0 || nnz < 0 || k <= 0 || !rowptr || (nnz > 0 && !colind))
    return fail(LAPIS_B200_ERR_ARG, "spmm plan: bad arguments");
  if ((rp_bytes != 4 && rp_bytes != 8) || (ci_bytes != 4 && ci_bytes != 8) || !valid_dtype(dtype))
    return fail(LAPIS_B200_ERR_ARG, "spmm plan: bad index width or dtype");
  if (ncols > 0x7fffffffLL) return fail(LAPIS_B200_ERR_UNSUPPORTED, "spmm plan: ncols >= 2^31");
  auto* p = new SpmmPlanImpl();
  p->nrows = nrows; p->ncols = ncols; p->nnz = nnz; p->k = k; p->dtype = dtype;
  cudaGetDevice(&p->device);
  const int64_t row_bytes = k * elem_bytes(dtype);
  if (hot_bytes < 0) hot_bytes = 0;
  // 16 MB measured best on config 3 (8.83 ms vs 9.40 without a plan, 8.99 at 32 MB,
  // 10.84 at 64 MB: a larger persisting set starves the streamed rest of L2)
  if (hot_bytes == 0) hot_bytes = 16ll << 20;
  const char* nohot = getenv("LAPIS_B200_SPMM_NOHOT");  // A/B runs: hints only
  if (nohot && nohot[0] == '1') hot_bytes = 0;
  int max_persist = 0;
  cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, p->device);
  cudaGetLastError();
  if (max_persist > 0 && hot_bytes > max_persist) hot_bytes = max_persist;
  const int64_t cap = hot_bytes > 0 ? std::min<int64_t>(ncols, hot_bytes / row_bytes) : 0;
  int rc = LAPIS_B200_OK;
  unsigned* counts = nullptr;
  int32_t* hot_index = nullptr;
  unsigned long long* hist = nullptr;  // [NB] then the slot counter
  constexpr int NB = 1 << 16;
  const int sms = num_sms();
  auto cleanup = [&]() {
    if (counts) cudaFreeAsync(counts, st);
    if (hot_index) cudaFreeAsync(hot_index, st);
    if (hist) cudaFreeAsync(hist, st);
  };
  rc = check_cuda(cudaMallocAsync((void**)&counts, (size_t)std::max<int64_t>(ncols, 1) * 4, st), "alloc(counts)");
  if (rc == LAPIS_B200_OK)
    rc = check_cuda(cudaMallocAsync((void**)&hot_index, (size_t)std::max<int64_t>(ncols, 1) * 4, st), "alloc(hot_index)");
  if (rc == LAPIS_B200_OK) rc = check_cuda(cudaMallocAsync((void**)&hist, (NB + 1) * 8, st), "alloc(hist)");
  if (rc == LAPIS_B200_OK) rc = check_cuda(cudaMallocAsync((void**)&p->colind_hot, (size_t)std::max<int64_t>(nnz, 1) * 4, st), "alloc(colind_hot)");
  if (rc == LAPIS_B200_OK && cap > 0) {
    rc = check_cuda(cudaMallocAsync((void**)&p->hot_cols, (size_t)cap * 4, st), "alloc(hot_cols)");
    if (rc == LAPIS_B200_OK)
      rc = check_cuda(cudaMallocAsync(&p->xhot, (size_t)cap * row_bytes, st), "alloc(xhot)");
  }
  if (rc == LAPIS_B200_OK) rc = check_cuda(cudaMemsetAsync(counts, 0, (size_t)std::max<int64_t>(ncols, 1) * 4, st), "memset");
  if (rc == LAPIS_B200_OK) rc = check_cuda(cudaMemsetAsync(hist, 0, (NB + 1) * 8, st), "memset");
  const int32_t* c32 = ci_bytes == 4 ? (const int32_t*)colind : nullptr;
  const int64_t* c64 = ci_bytes == 8 ? (const int64_t*)colind : nullptr;
  const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((nnz + 255) / 256, (int64_t)sms * 8));
  const unsigned gc = (unsigned)std::max<int64_t>(1, std::min<int64_t>((ncols + 255) / 256, (int64_t)sms * 8));
  if (rc == LAPIS_B200_OK && nnz > 0) {
    col_hist_kernel<<<g, 256, 0, st>>>(nnz, c32, c64, counts);
    rc = check_launch("col_hist_kernel");
  }
  if (rc == LAPIS_B200_OK) {
    count_hist_kernel<<<gc, 256, 0, st>>>(ncols, counts, hist, NB);
    rc = check_launch("count_hist_kernel");
  }
  std::vector<unsigned long long> h(NB, 0);
  if (rc == LAPIS_B200_OK)
    rc = check_cuda(cudaMemcpyAsync(h.data(), hist, NB * 8, cudaMemcpyDeviceToHost, st), "hist D2H");
  if (rc == LAPIS_B200_OK) rc = check_cuda(cudaStreamSynchronize(st), "plan sync");
  // threshold: the smallest count tau (>= 2: a row read once gains nothing)
  // whose columns with count >= tau fit the hot capacity
  unsigned tau = NB;
  {
    unsigned long long acc = 0;
    for (int v = NB - 1; v >= 2; --v) {
      if (acc + h[v] > (unsigned long long)cap) break;
      acc += h[v];
      tau = (unsigned)v;
    }
  }
  if (rc == LAPIS_B200_OK) rc = check_cuda(cudaMemsetAsync(hist + NB, 0, 8, st), "memset slot");
  if (rc == LAPIS_B200_OK) {
    hot_assign_kernel<<<gc, 256, 0, st>>>(ncols, counts, tau, cap, hist + NB, hot_index,
                                          p->hot_cols);
    rc = check_launch("hot_assign_kernel");
  }
  if (rc == LAPIS_B200_OK && nnz > 0) {
    hot_remap_kernel<<<g, 256, 0, st>>>(nnz, c32, c64, hot_index, p->colind_hot);
    rc = check_launch("hot_remap_kernel");
  }
  unsigned long long nh = 0;
  if (rc == LAPIS_B200_OK)
    rc = check_cuda(cudaMemcpyAsync(&nh, hist + NB, 8, cudaMemcpyDeviceToHost, st), "slot D2H");
  if (rc == LAPIS_B200_OK) rc = check_cuda(cudaStreamSynchronize(st), "plan sync");
  cleanup();
  if (rc != LAPIS_B200_OK) {
    if (p->colind_hot) cudaFree(p->colind_hot);
    if (p->hot_cols) cudaFree(p->hot_cols);
    if (p->xhot) cudaFree(p->xhot);
    delete p;
    return rc;
  }
  p->nhot = std::min<int64_t>((int64_t)nh, cap);
  // reuse hints, opt-in (LAPIS_B200_SPMM_HINT=1): needs column ids < 2^30 and
  // positions < 2^31.  Measured on config 3 with the 3-CTA HOT kernel: DRAM
  // 48.4 -> 46.3 GB per launch but 7.70 -> 7.96 ms (the policy branch costs
  // more than the traffic saves once the kernel runs at the copy rate)
  const char* he = getenv("LAPIS_B200_SPMM_HINT");
  if ((he && he[0] == '1') && nnz > 0 && nnz < 0x7fffffffLL && ncols < (1ll << 30)) {
    rc = spmm_reuse_hints(p, c32, c64, row_bytes, st);
    if (rc != LAPIS_B200_OK) {
      cudaFree(p->colind_hot);
      if (p->hot_cols) cudaFree(p->hot_cols);
      if (p->xhot) cudaFree(p->xhot);
      delete p;
      return rc;
    }
  }
  for (int v = (int)tau; v < NB && tau < (unsigned)NB; ++v) p->hot_entries += (int64_t)h[v] * v;
  // persisting L2 for the hot rows (process-wide limit; never lowered here)
  const size_t want = (size_t)p->nhot * row_bytes;
  const char* wenv = getenv("LAPIS_B200_SPMM_WINDOW");   // A/B runs: 0 = no persisting window
  if (want > 0 && max_persist > 0 && !(wenv && wenv[0] == '0')) {
    size_t cur = 0;
    cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
    if (cur < want) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min<size_t>(want, max_persist));
    cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
    p->window_bytes = std::min(cur, want);
    cudaGetLastError();
  }
  *out = p;
  return LAPIS_B200_OK;
}

int spmm_plan_info(void* plan, int64_t* out4) {
  auto* p = static_cast<SpmmPlanImpl*>(plan);
  if (!p || !out4) return fail(LAPIS_B200_ERR_ARG, "spmm plan info: null argument");
  out4[0] = p->nhot;
  out4[1] = p->hot_entries;
  out4[2] = (int64_t)p->window_bytes;
  out4[3] = p->nnz;
  return LAPIS_B200_OK;
}

int spmm_plan_hints(void* plan, int64_t* out_far) {
  auto* p = static_cast<SpmmPlanImpl*>(plan);
  if (!p || !out_far) return fail(LAPIS_B200_ERR_ARG, "spmm plan hints: null argument");
  *out_far = p->hints ? p->far_entries : -1;
  return LAPIS_B200_OK;
}

int spmm_plan_destroy(void* plan) {
  auto* p = static_cast<SpmmPlanImpl*>(plan);
  if (!p) return LAPIS_B200_OK;
  cudaFree(p->colind_hot);
  if (p->hot_cols) cudaFree(p->hot_cols);
  if (p->xhot) cudaFree(p->xhot);
  if (p->window_bytes) cudaCtxResetPersistingL2Cache();
  delete p;
  return check_cuda(cudaGetLastError(), "spmm plan destroy");
}

int spmm_csr_plan(void* plan, const void* rowptr, int rp_bytes, const void* colind, int ci_bytes,
                  const void* values, const void* X, int64_t ldx, void* Y, int64_t ldy, int dtype,
                  cudaStream_t st) {
  auto* p = static_cast<SpmmPlanImpl*>(plan);
  if (!p) return fail(LAPIS_B200_ERR_ARG, "spmm: null plan");
  if (dtype != p->dtype) return fail(LAPIS_B200_ERR_ARG, "spmm plan: dtype differs from the plan's");
  const int64_t nrows = p->nrows, nnz = p->nnz, k = p->k;
  if ((rp_bytes != 4 && rp_bytes != 8) || (ci_bytes != 4 && ci_bytes != 8))
    return fail(LAPIS_B200_ERR_ARG, "spmm: index widths must be 4 or 8 bytes");
  if (ldx < k || ldy < k) return fail(LAPIS_B200_ERR_ARG, "spmm: leading dimension < k");
  if (!rowptr || (nrows > 0 && !Y) || (nnz > 0 && (!colind || !values || !X)))
    return fail(LAPIS_B200_ERR_ARG, "spmm: null operand");
  if (nrows == 0) return LAPIS_B200_OK;
  const int64_t row_bytes = k * elem_bytes(dtype);
  HotMap hm{p->colind_hot, p->xhot, k};
  if (p->nhot > 0) {
    const int sms = num_sms();
    const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((p->nhot + 7) / 8, (int64_t)sms * 8));
    hot_gather_kernel<<<g, 256, 0, st>>>(p->nhot, row_bytes, p->hot_cols, (const unsigned char*)X,
                                         ldx * elem_bytes(dtype), (unsigned char*)p->xhot);
    LB_TRY(check_launch("hot_gather_kernel"));
  }
  const bool window = p->window_bytes > 0;
  if (window) {
    cudaStreamAttrValue a = {};
    a.accessPolicyWindow.base_ptr = p->xhot;
    a.accessPolicyWindow.num_bytes = (size_t)p->nhot * row_bytes;
    a.accessPolicyWindow.hitRatio =
        (float)std::min(1.0, (double)p->window_bytes / (double)a.accessPolicyWindow.num_bytes);
    a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &a);
    cudaGetLastError();
  }
  const HotMap* hp = (p->nhot > 0 || p->hints) ? &hm : nullptr;
  int rc;
#define LB_SPMMP(T)                                                                              \
  if (rp_bytes == 8 && ci_bytes == 4) rc = SpmmOp<T, int64_t, int32_t>::run(nrows, nnz, k, rowptr, colind, values, X, ldx, Y, ldy, st, nullptr, hp); \
  else if (rp_bytes == 8) rc = SpmmOp<T, int64_t, int64_t>::run(nrows, nnz, k, rowptr, colind, values, X, ldx, Y, ldy, st, nullptr, hp); \
  else if (ci_bytes == 4) rc = SpmmOp<T, int32_t, int32_t>::run(nrows, nnz, k, rowptr, colind, values, X, ldx, Y, ldy, st, nullptr, hp); \
  else rc = SpmmOp<T, int32_t, int64_t>::run(nrows, nnz, k, rowptr, colind, values, X, ldx, Y, ldy, st, nullptr, hp);
  switch (dtype) {
    case LAPIS_B200_F64: { LB_SPMMP(double) break; }
    case LAPIS_B200_F32: { LB_SPMMP(float) break; }
    case LAPIS_B200_I64: { LB_SPMMP(long long) break; }
    default: { LB_SPMMP(int) break; }
  }
#undef LB_SPMMP
  if (window) {
    cudaStreamAttrValue a = {};
    a.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &a);
    cudaGetLastError();
  }
  return rc;
}

}  // namespace lapis_b200
