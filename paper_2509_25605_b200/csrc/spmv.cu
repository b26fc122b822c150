// spmv.cu — CSR SpMV for sm_100a.
//
// Semantics: interp.py:798-812 (_h_spmv_csr) — y[i] = sum over
// j in [rowptr[i], max(rowptr[i], rowptr[i+1])) of values[j] * x[colind[j]],
// ascending j, each op rounded (interp.py:168-183).
//
// Two kernels:
//
// 1. spmv_tile_kernel (default, vector_length = 0): a "row-stream tile".
//    Work units are rows + nonzeros (key(r) = rowptr[r] - rowptr[0] + r is
//    strictly increasing); tile c owns the rows whose key falls in
//    [c*TILE_KEYS, (c+1)*TILE_KEYS), so every tile holds a bounded number of
//    rows AND nonzeros whatever the row-length distribution (empty rows and
//    hub rows included).  The CTA streams its contiguous nonzero range with
//    16-byte loads (colind, values), gathers x through the read-only path,
//    stages the products in shared memory, and then ONE thread per row sums
//    that row's products in ascending order with non-contracted mul/add: the
//    result is bit-identical to the reference for every row of <= LONG_ROW
//    entries.  A longer row can only be the last row of its tile; it is
//    reduced by the whole CTA (strided partials + fixed tree).
//    The tile -> first-row table is a structure-only plan (partition kernel),
//    computed per call or cached in a lapis_b200_csr_plan.
//
// 2. spmv_vector_kernel<VL> (vector_length = VL): the emitted TeamPolicy
//    mapping of golden/cpp/spmv.hpp:45-66 — one row per VL lanes
//    (Kokkos thread -> sub-warp, vector -> lane), ThreadVectorRange reduce as
//    a shuffle tree, single(PerThread) store by lane 0.
//
// 3. spmv_warpblock_kernel (plans of regular, monotone, short-row structures):
//    32 rows per warp, their contiguous entry range streamed with coalesced
//    loads into a warp-private shared-memory window, each lane folding its own
//    row in ascending order (bit-identical).
#include "common.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <cstdio>

namespace lapis_b200 {

constexpr int TILE_KEYS = 1024;                   // rows + nonzeros owned per tile (plan grain)
constexpr int LONG_ROW = 512;                     // last-row length handled in shared memory
constexpr int TILE_CAP = TILE_KEYS + LONG_ROW;    // products staged per tile
// plan: mean row length below which the warp-block kernel is chosen by default.
// 0 = never: measured on B200 (C1 5-point: 35.7 us vs 30.1 us for the VL = 1
// vector kernel; C5 exact mode 4.35 vs 4.27 TB/s), so it is only selected by
// LAPIS_B200_SPMV_KERNEL=wb
constexpr double WARPBLOCK_MAX_MEAN = 0.0;

// Device-side kernel choice for calls without a plan (lapis_b200_spmv_csr,
// vector_length = 0): a stats pass writes {longest row, descending flag};
// the regular-structure kernel and the tile kernel are both launched and each
// returns at once unless the stats select it (no host round trip).
struct RowGuard {
  const unsigned long long* stats = nullptr;  // nullptr: no guard
  long long thresh = 0;                       // regular iff monotone && max_len <= thresh
  int want = 0;  // 1 regular, 2 monotone irregular, 3 non-monotone
};
__device__ __forceinline__ bool row_guard_skip(const RowGuard& g) {
  if (!g.stats) return false;
  const bool monotone = g.stats[1] == 0;
  const int cls = !monotone ? 3 : ((long long)g.stats[0] <= g.thresh ? 1 : 2);
  return cls != g.want;
}

// ---------------------------------------------------------------- plan
// tile_row[c]  = first row owned by tile c (c in [0, ntiles]; tile_row[ntiles] = nrows)
// tile_nnz[c]  = rowptr[tile_row[c]] (absolute), so a tile can start streaming
//                its nonzeros without first reading rowptr
template <class RP>
__global__ void tile_partition_kernel(int64_t nrows, const RP* __restrict__ rowptr,
                                      int64_t ntiles, int64_t* __restrict__ tile_row,
                                      int64_t* __restrict__ tile_nnz, RowGuard guard = RowGuard()) {
  if (row_guard_skip(guard)) return;
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r > nrows) return;
  const int64_t base = (int64_t)rowptr[0];
  const int64_t rp = (int64_t)rowptr[r];
  const int64_t key = rp - base + r;
  const int64_t keyprev = (r == 0) ? -1 : (int64_t)rowptr[r - 1] - base + (r - 1);
  // tile c starts at row r iff c*TILE_KEYS lies in (keyprev, key]
  const int64_t c0 = (keyprev < 0) ? 0 : keyprev / TILE_KEYS + 1;
  const int64_t c1 = (r == nrows) ? ntiles : key / TILE_KEYS;
  for (int64_t c = c0; c <= c1 && c <= ntiles; ++c) {
    tile_row[c] = r;
    tile_nnz[c] = rp;
  }
}

// ------------------------------------------------------------ vector loads
template <class T>
__device__ __forceinline__ void load4(const T* p, T out[4]) {
  if constexpr (sizeof(T) == 4) {
    int4 v = ld_stream(reinterpret_cast<const int4*>(p));
    const int w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) memcpy(&out[q], &w[q], 4);
  } else {
    longlong2 a = ld_stream(reinterpret_cast<const longlong2*>(p));
    longlong2 b = ld_stream(reinterpret_cast<const longlong2*>(p + 2));
    const long long w[4] = {a.x, a.y, b.x, b.y};
#pragma unroll
    for (int q = 0; q < 4; ++q) memcpy(&out[q], &w[q], 8);
  }
}

template <class T, int NT>
__device__ __forceinline__ T block_sum(T part, T* scratch) {
  // fixed-order tree: xor butterfly inside each warp, then thread 0 folds the
  // per-warp partials in ascending warp order
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) part = Arith<T>::add(part, shfl_xor(part, off));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) scratch[warp] = part;
  __syncthreads();
  T tot = Arith<T>::zero();
  if (threadIdx.x == 0)
    for (int w = 0; w < NT / 32; ++w) tot = Arith<T>::add(tot, scratch[w]);
  return tot;
}

// long row (> LONG_ROW entries) owned by this CTA.  fp64 / ints: strided
// partials + fixed tree (ints are order-independent; fp64 stays far inside the
// 1e-12 contract).  fp32: the reference's exact sequential order — products
// staged chunk by chunk, thread 0 folds them in ascending order — because a
// reassociated fp32 sum of thousands of terms can differ from the reference's
// own rounding by more than 1e-5.
template <class T, class CI, int NT>
__device__ void long_row(int64_t rs, int64_t e, const CI* __restrict__ colind,
                         const T* __restrict__ values, const T* __restrict__ x, T* prod,
                         T* scratch, T* __restrict__ yout) {
  if constexpr (sizeof(T) == 4 && !std::is_integral<T>::value) {
    T acc = Arith<T>::zero();
    for (int64_t c0 = rs; c0 < e; c0 += TILE_CAP) {
      const int64_t c1 = (c0 + TILE_CAP < e) ? c0 + TILE_CAP : e;
      __syncthreads();
      for (int64_t j = c0 + threadIdx.x; j < c1; j += NT)
        prod[j - c0] = Arith<T>::mul(values[j], __ldg(x + (int64_t)colind[j]));
      __syncthreads();
      if (threadIdx.x == 0)
        for (int64_t j = 0; j < c1 - c0; ++j) acc = Arith<T>::add(acc, prod[j]);
    }
    if (threadIdx.x == 0) *yout = acc;
  } else {
    T part = Arith<T>::zero();
#pragma unroll 4
    for (int64_t j = rs + threadIdx.x; j < e; j += NT)
      part = Arith<T>::add(part, Arith<T>::mul(values[j], __ldg(x + (int64_t)colind[j])));
    T tot = block_sum<T, NT>(part, scratch);
    if (threadIdx.x == 0) *yout = tot;
  }
}

// ------------------------------------------------------------ tile kernel
// Persistent: CTA b processes tiles b, b + G, b + 2G, ... (G = gridDim.x).
// Three things overlap in every iteration `it`:
//   * the TMA engine streams the nonzeros (colind, values; 16-byte aligned
//     cp.async.bulk into a ST-deep shared-memory ring, one mbarrier per stage)
//     of tiles it+2 .. it+ST;
//   * the x gathers of tile it+1 (read-only path, registers) are in flight;
//   * tile it's rows are summed sequentially from its staged products.
// Thread 0 prefetches the plan of tile it+ST into registers at the top of the
// iteration and refills tile it's stage at the bottom.
template <class T, class CI, int ST>
struct StreamSmem {
  static constexpr int CI_ELEMS = TILE_CAP + 16 / sizeof(CI) * 2;  // + alignment slack
  static constexpr int V_ELEMS = TILE_CAP + 16 / sizeof(T) * 2;
  static constexpr size_t CI_BYTES = (CI_ELEMS * sizeof(CI) + 127) / 128 * 128;
  static constexpr size_t V_BYTES = (V_ELEMS * sizeof(T) + 127) / 128 * 128;
  static constexpr size_t STAGE_BYTES = CI_BYTES + V_BYTES;
  static constexpr size_t TOTAL = ST * STAGE_BYTES;
};

template <class T, class RP, class CI, int NT, int ST>
__global__ void __launch_bounds__(NT)
spmv_tile_kernel(const RP* __restrict__ rowptr, const CI* __restrict__ colind,
                 const T* __restrict__ values, const T* __restrict__ x, T* __restrict__ y,
                 const int64_t* __restrict__ tile_row, const int64_t* __restrict__ tile_nnz,
                 int64_t ntiles, int tma_ok, RowGuard guard = RowGuard()) {
  if (row_guard_skip(guard)) return;
  using L = StreamSmem<T, CI, ST>;
  constexpr int PER = (TILE_CAP + NT - 1) / NT;        // streamed entries per thread
  constexpr int RPER = (TILE_KEYS + NT - 1) / NT;      // owned rows per thread
  constexpr int64_t CA = 16 / sizeof(CI), VA = 16 / sizeof(T);
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t full[ST];
  __shared__ int64_t meta[ST][4];            // r_begin, r_end, s, e
  __shared__ int32_t moff[ST][3];            // colind offset, values offset, direct flag
  __shared__ int32_t rps[2][TILE_KEYS + 1];  // row starts relative to s (double-buffered)
  __shared__ T scratch[NT / 32];
  const int tid = threadIdx.x;
  auto sci = [&](int st) { return reinterpret_cast<CI*>(smem + st * L::STAGE_BYTES); };
  auto sv = [&](int st) { return reinterpret_cast<T*>(smem + st * L::STAGE_BYTES + L::CI_BYTES); };

  // the streams end at rowptr[nrows]; an aligned-up bulk copy must not pass it
  const int64_t nnz_end = tid == 0 ? tile_nnz[ntiles] : 0;
  // thread 0 only: put tile (rb, re, s0, e0) in flight on stage `st`
  auto issue = [&](int st, int64_t rb, int64_t re, int64_t s0, int64_t e0) {
    const int64_t et = (e0 - s0 > TILE_CAP) ? s0 + TILE_CAP : e0;
    const int64_t sc = s0 & ~(CA - 1), ec = (et + CA - 1) & ~(CA - 1);
    const int64_t sv0 = s0 & ~(VA - 1), ev = (et + VA - 1) & ~(VA - 1);
    const bool direct = !tma_ok || re <= rb || et <= s0 || ec > nnz_end || ev > nnz_end;
    meta[st][0] = rb; meta[st][1] = re; meta[st][2] = s0; meta[st][3] = e0;
    moff[st][0] = direct ? 0 : (int32_t)(s0 - sc);
    moff[st][1] = direct ? 0 : (int32_t)(s0 - sv0);
    moff[st][2] = direct;
    if (direct) {
      mbar_arrive(&full[st]);
    } else {
      const uint32_t bc = (uint32_t)((ec - sc) * sizeof(CI)), bv = (uint32_t)((ev - sv0) * sizeof(T));
      mbar_arrive_expect_tx(&full[st], bc + bv);
      bulk_g2s(sci(st), colind + sc, bc, &full[st]);
      bulk_g2s(sv(st), values + sv0, bv, &full[st]);
    }
  };

  // gather state of the tile being prepared (held across the row sums of the previous one)
  T xg[PER];
  int64_t rpv[RPER];
  // stage A: wait for tile `k`'s stream, issue its x gathers and rowptr loads
  auto gather = [&](int64_t k) {
    const int st = (int)(k % ST);
    const uint32_t parity = (uint32_t)((k / ST) & 1);
    const int64_t rb = meta[st][0], re = meta[st][1], s0 = meta[st][2], e0 = meta[st][3];
    const int nr = (int)(re - rb);
#pragma unroll
    for (int u = 0; u < RPER; ++u) {
      const int i = tid + u * NT;
      rpv[u] = i < nr ? (int64_t)rowptr[rb + i] : 0;
    }
    mbar_wait(&full[st], parity);
    const int n = nr > 0 ? (int)(((e0 - s0 > TILE_CAP) ? TILE_CAP : e0 - s0)) : 0;
    const int dc = moff[st][0], direct = moff[st][2];
    const CI* cbuf = sci(st) + dc;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int q = tid + u * NT;
      int64_t col = 0;
      if (q < n) col = direct ? (int64_t)colind[s0 + q] : (int64_t)cbuf[q];
      xg[u] = q < n ? __ldg(x + col) : T(0);
    }
  };
  // stage C: products of tile `k` in place (values slot) and its row starts
  auto finish = [&](int64_t k) {
    const int st = (int)(k % ST);
    const int64_t rb = meta[st][0], re = meta[st][1], s0 = meta[st][2], e0 = meta[st][3];
    const int nr = (int)(re - rb);
    const int n = nr > 0 ? (int)(((e0 - s0 > TILE_CAP) ? TILE_CAP : e0 - s0)) : 0;
    const int dv = moff[st][1], direct = moff[st][2];
    T* prod = sv(st) + dv;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int q = tid + u * NT;
      if (q < n) prod[q] = Arith<T>::mul(direct ? values[s0 + q] : prod[q], xg[u]);
    }
    int32_t* rp = rps[k & 1];
#pragma unroll
    for (int u = 0; u < RPER; ++u) {
      const int i = tid + u * NT;
      if (i < nr) {
        const int64_t v = rpv[u] - s0;
        rp[i] = (int32_t)(v < TILE_CAP ? v : TILE_CAP);
      }
    }
  };
  // stage B: sequential row sums of tile `k` (reference order), long last row
  auto rows = [&](int64_t k) {
    const int st = (int)(k % ST);
    const int64_t rb = meta[st][0], re = meta[st][1], s0 = meta[st][2], e0 = meta[st][3];
    const int nr = (int)(re - rb);
    if (nr <= 0) return;
    const int32_t* rp = rps[k & 1];
    T* prod = sv(st) + moff[st][1];
    const int64_t last_b = rp[nr - 1];
    const bool long_last = (e0 - s0) - last_b > LONG_ROW;
    const int nshort = long_last ? nr - 1 : nr;
    for (int i = tid; i < nshort; i += NT) {
      int q = rp[i];
      const int end = (i + 1 < nr) ? rp[i + 1] : (int)(e0 - s0);
      T acc = Arith<T>::zero();
      for (; q + 4 <= end; q += 4) {
        const T p0 = prod[q], p1 = prod[q + 1], p2 = prod[q + 2], p3 = prod[q + 3];
        acc = Arith<T>::add(acc, p0);
        acc = Arith<T>::add(acc, p1);
        acc = Arith<T>::add(acc, p2);
        acc = Arith<T>::add(acc, p3);
      }
      for (; q < end; ++q) acc = Arith<T>::add(acc, prod[q]);
      y[rb + i] = acc;
    }
    if (long_last) long_row<T, CI, NT>(s0 + last_b, e0, colind, values, x, prod, scratch, y + re - 1);
  };

  if (tid == 0) {
    for (int st = 0; st < ST; ++st) mbar_init(&full[st], 1);
    fence_barrier_init();
    for (int st = 0; st < ST; ++st) {
      const int64_t c = blockIdx.x + (int64_t)st * gridDim.x;
      if (c < ntiles) issue(st, tile_row[c], tile_row[c + 1], tile_nnz[c], tile_nnz[c + 1]);
    }
  }
  __syncthreads();
  if ((int64_t)blockIdx.x < ntiles) {
    gather(0);
    finish(0);
  }
  __syncthreads();

  for (int64_t it = 0;; ++it) {
    const int64_t c = blockIdx.x + it * gridDim.x;
    if (c >= ntiles) break;
    const int64_t cn = c + (int64_t)ST * gridDim.x;   // tile refilled at the bottom
    int64_t p0 = 0, p1 = 0, p2 = 0, p3 = 0;
    if (tid == 0 && cn < ntiles) { p0 = tile_row[cn]; p1 = tile_row[cn + 1]; p2 = tile_nnz[cn]; p3 = tile_nnz[cn + 1]; }
    const bool has_next = c + gridDim.x < ntiles;
    if (has_next) gather(it + 1);   // A: gathers of tile it+1 in flight
    rows(it);                       // B: row sums of tile it
    if (has_next) finish(it + 1);   // C: products of tile it+1
    __syncthreads();
    if (tid == 0 && cn < ntiles) {
      fence_proxy_async();
      issue((int)(it % ST), p0, p1, p2, p3);
    }
  }
}

// ---------------------------------------------------------- vector kernel
// One row per VL lanes (Kokkos thread -> sub-warp, vector -> lane), row groups
// walked grid-stride with a warp-uniform trip count.
//   EXACT = false: the emitted TeamPolicy mapping (golden/cpp/spmv.hpp:45-66):
//     lane-strided partials, ThreadVectorRange reduce as a shuffle tree.
//   EXACT = true: same load pattern, but each step's VL products (entries
//     j0 .. j0+VL-1) are folded into the accumulator in ascending j through
//     in-group shuffles, so the row sum is the reference's sequential sum bit
//     for bit (out-of-row lanes contribute +0.0, which leaves any accumulator
//     that can arise unchanged: the running sum starts at +0.0 and can never
//     become -0.0).  Two steps are unrolled to keep 2*VL loads per row in flight.
template <class T, class RP, class CI, int VL, bool EXACT>
__global__ void __launch_bounds__(256)
spmv_vector_kernel(int64_t nrows, const RP* __restrict__ rowptr, const CI* __restrict__ colind,
                   const T* __restrict__ values, const T* __restrict__ x, T* __restrict__ y,
                   RowGuard guard = RowGuard()) {
  // launched with programmatic stream serialization (one-wave problems): wait
  // for the previous grid's completion before any memory access, and let
  // the next grid's CTAs launch as soon as this grid's have all started
  // (no-ops for a plain launch)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (row_guard_skip(guard)) return;
  const int lane = threadIdx.x & (VL - 1);
  const unsigned gmask = (VL == 32) ? 0xffffffffu
                                    : (((1u << VL) - 1u) << ((threadIdx.x & 31) & ~(VL - 1)));
  const int64_t groups_per_grid = (int64_t)gridDim.x * (blockDim.x / VL);
  const int64_t warp_first = ((int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) / VL;
  const int64_t my_off = (threadIdx.x & 31) / VL;
  for (int64_t wrow = warp_first; wrow < nrows; wrow += groups_per_grid) {
    const int64_t row = wrow + my_off;
    T acc = Arith<T>::zero();
    if (row < nrows) {
      const int64_t b = (int64_t)rowptr[row];
      int64_t e = (int64_t)rowptr[row + 1];
      if (e < b) e = b;  // interp.py:808 range(begin, max(begin, end))
      if constexpr (EXACT) {
        int64_t j0 = b;
        for (; j0 + VL < e; j0 += 2 * VL) {
          const int64_t ja = j0 + lane, jb = j0 + VL + lane;
          const T pa = Arith<T>::mul(values[ja], __ldg(x + (int64_t)colind[ja]));
          const T pb = jb < e ? Arith<T>::mul(values[jb], __ldg(x + (int64_t)colind[jb])) : T(0);
#pragma unroll
          for (int s2 = 0; s2 < VL; ++s2)
            acc = Arith<T>::add(acc, VL == 1 ? pa : __shfl_sync(gmask, pa, s2, VL));
#pragma unroll
          for (int s2 = 0; s2 < VL; ++s2)
            acc = Arith<T>::add(acc, VL == 1 ? pb : __shfl_sync(gmask, pb, s2, VL));
        }
        if (j0 < e) {
          const int64_t ja = j0 + lane;
          const T pa = ja < e ? Arith<T>::mul(values[ja], __ldg(x + (int64_t)colind[ja])) : T(0);
#pragma unroll
          for (int s2 = 0; s2 < VL; ++s2)
            acc = Arith<T>::add(acc, VL == 1 ? pa : __shfl_sync(gmask, pa, s2, VL));
        }
      } else {
        for (int64_t j = b + lane; j < e; j += VL)
          acc = Arith<T>::add(acc, Arith<T>::mul(values[j], __ldg(x + (int64_t)colind[j])));
      }
    }
    if constexpr (!EXACT) {
#pragma unroll
      for (int off = VL / 2; off >= 1; off >>= 1) acc = Arith<T>::add(acc, shfl_xor(acc, off, VL));
    }
    if (lane == 0 && row < nrows) y[row] = acc;
  }
}

// ------------------------------------------------------- warp-block kernel
// A warp owns 32 consecutive rows, whose entries form ONE contiguous range
// [rowptr[r0], rowptr[r0+32]) when rowptr is monotone (the plan checks).  The
// range is streamed in rounds of 32*U entries: each lane issues U coalesced
// colind/values loads and U x gathers up front (all independent, so a warp has
// 3U loads in flight), stores the products in a warp-private shared-memory
// window, and then each lane folds ITS row's products of the window in
// ascending j.  Every row sum is therefore the reference's sequential sum bit
// for bit (interp.py:808-811), whatever the row lengths, while every global
// load instruction reads 32 consecutive entries.  Short regular rows (C1: 5
// per row) are the case the vector kernel serves worst: one row per lane there
// reads 5 strided entries with about 2 loads in flight per thread.
// Schedulable (non-volatile) read-only load with an L2 eviction policy.
template <class T> __device__ __forceinline__ T ld_pol(const T* p, uint64_t pol);
template <> __device__ __forceinline__ double ld_pol<double>(const double* p, uint64_t pol) {
  double v; asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol)); return v;
}
template <> __device__ __forceinline__ float ld_pol<float>(const float* p, uint64_t pol) {
  float v; asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol)); return v;
}
template <> __device__ __forceinline__ long long ld_pol<long long>(const long long* p, uint64_t pol) {
  long long v; asm("ld.global.nc.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol)); return v;
}
template <> __device__ __forceinline__ long ld_pol<long>(const long* p, uint64_t pol) {
  long v; asm("ld.global.nc.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol)); return v;
}
template <> __device__ __forceinline__ int ld_pol<int>(const int* p, uint64_t pol) {
  int v; asm("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol)); return v;
}

// POL: the structure stream (each 128-B line consumed whole by one coalesced
// warp load) is read L2::evict_first and the x gathers L2::evict_last, so x
// (80 MB for config 3's 10M rows) stays in the 126 MB L2 instead of being
// pushed out by the 1.2 GB entry stream.
// (three CTAs per SM at U = 16 — 80 registers — measured 1.84 vs 1.09 ms)
template <class T, class RP, class CI, int U, bool EXACT, bool POL = false>
__global__ void __launch_bounds__(256)
spmv_warpblock_kernel(int64_t nrows, const RP* __restrict__ rowptr, const CI* __restrict__ colind,
                      const T* __restrict__ values, const T* __restrict__ x, T* __restrict__ y,
                      unsigned long long* __restrict__ next, RowGuard guard = RowGuard()) {
  if (row_guard_skip(guard)) return;
  uint64_t pol_first = 0, pol_last = 0;
  if constexpr (POL) {
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_last));
  }
  constexpr int CAP = 32 * U;
  __shared__ T win[8][CAP];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T* __restrict__ my = win[w];
  const int64_t nblk = (nrows + 31) >> 5;
  const int64_t stride = (int64_t)gridDim.x * 8;
  // blocks of 32 rows from a per-call counter when given (irregular rows: a
  // static split leaves SMs idle behind their slowest warp), else grid-stride
  auto grab = [&]() -> int64_t {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(next, 1ull);
    return (int64_t)__shfl_sync(0xffffffffu, t, 0);
  };
  for (int64_t blk = next ? grab() : (int64_t)blockIdx.x * 8 + w; blk < nblk;
       blk = next ? grab() : blk + stride) {
    const int64_t row = (blk << 5) + lane;
    const int64_t last = min(nrows, (blk << 5) + 32);
    int64_t b = 0, e = 0;
    if (row < nrows) {
      b = (int64_t)rowptr[row];
      e = (int64_t)rowptr[row + 1];
    }
    const int64_t lo = __shfl_sync(0xffffffffu, b, 0);
    const int64_t hi = (int64_t)rowptr[last];  // one line, shared by the warp
    if (row >= nrows) b = e = hi;
    T acc = Arith<T>::zero();
    for (int64_t base = lo; base < hi; base += CAP) {
      CI c[U];
      T v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t j = base + u * 32 + lane;
        if constexpr (POL) {
          c[u] = j < hi ? ld_pol<CI>(colind + j, pol_first) : CI(0);
          v[u] = j < hi ? ld_pol<T>(values + j, pol_first) : T(0);
        } else {
          c[u] = j < hi ? colind[j] : CI(0);
          v[u] = j < hi ? values[j] : T(0);
        }
      }
      T p[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t j = base + u * 32 + lane;
        if constexpr (POL)
          p[u] = j < hi ? ld_pol<T>(x + (int64_t)c[u], pol_last) : T(0);
        else
          p[u] = j < hi ? __ldg(x + (int64_t)c[u]) : T(0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) my[u * 32 + lane] = Arith<T>::mul(v[u], p[u]);
      __syncwarp();
      const int64_t s = max(b, base), t = min(e, base + CAP);
      if constexpr (EXACT) {
        for (int64_t j = s; j < t; ++j) acc = Arith<T>::add(acc, my[j - base]);
      } else {
        // a row's segment of more than 32 products in this window (a hub row)
        // is folded by the whole warp — lane-strided partials, fixed xor
        // tree, added to the owner's sum in window order (deterministic, the
        // ThreadVectorRange reduce); shorter segments by their own lane in order
        // (rows of <= LONG_ROW entries always fold in order: bit-identical,
        // the tile kernel's contract)
        const bool coop = (t - s > 32) && (e - b > LONG_ROW);
        unsigned big = __ballot_sync(0xffffffffu, coop);
        while (big) {
          const int owner = __ffs(big) - 1;
          big &= big - 1;
          const int64_t os = __shfl_sync(0xffffffffu, s, owner);
          const int64_t ot = __shfl_sync(0xffffffffu, t, owner);
          T part = Arith<T>::zero();
          for (int64_t j = os + lane; j < ot; j += 32) part = Arith<T>::add(part, my[j - base]);
#pragma unroll
          for (int off = 16; off >= 1; off >>= 1) part = Arith<T>::add(part, shfl_xor(part, off));
          if (lane == owner) acc = Arith<T>::add(acc, part);
        }
        if (!coop)
          for (int64_t j = s; j < t; ++j) acc = Arith<T>::add(acc, my[j - base]);
      }
      __syncwarp();
    }
    if (row < nrows) y[row] = acc;
  }
}

// ------------------------------------------------------- row-stream kernel
// Exact (reference-order) SpMV for regular structures, one row per thread.
// A tile is NT consecutive rows; their contiguous entry range is brought into
// a ST-deep shared-memory ring by the TMA engine (cp.async.bulk of colind and
// values, one mbarrier per stage), so no thread waits on the structure stream
// and every DRAM byte of it moves in 16-byte-aligned bulk transfers.  Thread
// i folds row r0+i sequentially — colind from shared memory, the x gather
// (lanes hold consecutive rows: for stencils the 32 gathers of one
// instruction are consecutive x entries), the product, the ordered add — in
// chunks of MC entries whose gathers are all issued before the chunk's adds.
// Small tiles (NT = 64: 21.5 KB per stage for 27-point rows) give five
// independent CTA pipelines per SM, each with a tile in flight while the
// previous one folds.  The row sum is the reference's sequential sum bit for
// bit (interp.py:808-811) whatever the row lengths.  A tile whose entries
// exceed the stage (irregular rows), or the unaligned tail of the last tile,
// is read from global memory directly; so is a row whose range lies outside
// its tile's stream (a decreasing rowptr), clamped to range(begin,
// max(begin, end)) (interp.py:808).  Shared-memory reads: lane i reads entry
// b_i + u, b_i = i * len — conflict-free for odd row lengths (27-point).
template <class T, class CI, class RP, int NT, int CAP, int ST>
struct RowStreamSmem {
  static constexpr int CA = 16 / sizeof(CI), VA = 16 / sizeof(T);
  static constexpr int RP_N = NT + 16 / (int)sizeof(RP);  // the tile's NT + 1 row offsets, 16-byte multiple
  static constexpr size_t CI_BYTES = ((CAP + CA) * sizeof(CI) + 127) / 128 * 128;
  static constexpr size_t V_BYTES = ((CAP + VA) * sizeof(T) + 127) / 128 * 128;
  static constexpr size_t RP_BYTES = (RP_N * sizeof(RP) + 127) / 128 * 128;
  static constexpr size_t STAGE_BYTES = CI_BYTES + V_BYTES + RP_BYTES;
  static constexpr size_t TOTAL = ST * STAGE_BYTES;
};

// one row's ordered sum: chunks of MC entries, each chunk's gathers issued
// before its adds; cp / vp point at the row's first entry (shared or global)
template <class T, class CI, int MC>
__device__ __forceinline__ T row_fold(const CI* __restrict__ cp, const T* __restrict__ vp, int n,
                                      const T* __restrict__ x) {
  T acc = Arith<T>::zero();
  for (int q = 0; q < n; q += MC) {
    int64_t c[MC];
#pragma unroll
    for (int u = 0; u < MC; ++u) c[u] = q + u < n ? (int64_t)cp[q + u] : 0;
    T xv[MC];
#pragma unroll
    for (int u = 0; u < MC; ++u) xv[u] = ld_ord<T>(x + c[u], q + u < n);
#pragma unroll
    for (int u = 0; u < MC; ++u)
      if (q + u < n) acc = Arith<T>::add(acc, Arith<T>::mul(vp[q + u], xv[u]));
  }
  return acc;
}

// per-CTA start / end timestamps and SM id (LAPIS_B200_RS_TIMES=<file>: a
// tuning aid for the static tile split; off by default)
__device__ int g_rs_dbg = 0;
__device__ unsigned long long g_rs_times[3 * 4096];
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <class T, class RP, class CI, int NT, int CAP, int ST, int MC>
__global__ void __launch_bounds__(NT)
spmv_rowstream_kernel(int64_t nrows, const RP* __restrict__ rowptr, const CI* __restrict__ colind,
                      const T* __restrict__ values, const T* __restrict__ x, T* __restrict__ y,
                      int tma_ok, int64_t nstatic, unsigned long long* __restrict__ next_tile,
                      int chunk, RowGuard guard = RowGuard()) {
  if (row_guard_skip(guard)) return;
  const bool dbg = g_rs_dbg && blockIdx.x < 4096;
  unsigned long long t_start = dbg ? global_ns() : 0;
  constexpr int ROWS = NT;
  using L = RowStreamSmem<T, CI, RP, NT, CAP, ST>;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t full[ST];
  // per stage: first staged entry of colind / values (aligned down; -1:
  // direct), the tile (-1: none left), its entry range, rowptr slice staged
  __shared__ int64_t meta[ST][6];
  const int tid = threadIdx.x;
  const int gi = tid;
  const int64_t ntiles = (nrows + ROWS - 1) / ROWS;
  const int64_t G = gridDim.x;
  auto sci = [&](int st) { return reinterpret_cast<CI*>(smem + st * L::STAGE_BYTES); };
  auto sv = [&](int st) { return reinterpret_cast<T*>(smem + st * L::STAGE_BYTES + L::CI_BYTES); };
  auto srp = [&](int st) {
    return reinterpret_cast<RP*>(smem + st * L::STAGE_BYTES + L::CI_BYTES + L::V_BYTES);
  };
  const int64_t nnz_end = tid == 0 ? (int64_t)rowptr[nrows] : 0;
  // tiles [0, nstatic): CTA b takes b, b + G, ... in order; tiles [nstatic,
  // ntiles) are handed out by the atomic counter, so a CTA that fell behind
  // (x gathers no longer hitting the L2 the other CTAs keep warm) takes fewer
  // (thread 0 claims runs of `chunk` consecutive counter tiles, each run one
  // run ahead of its use, so the atomic's round trip overlaps the folds)
  int64_t next_static = blockIdx.x;  // thread 0's next static tile
  int64_t claimed = -1;              // thread 0's next run, claimed ahead
  int64_t cur = 0, cur_end = 0;      // thread 0's current run
  auto claim = [&]() -> int64_t {
    return next_tile ? nstatic + (int64_t)atomicAdd(next_tile, 1ull) * chunk : ntiles;
  };
  auto next_id = [&]() -> int64_t {
    if (next_static < nstatic) {
      const int64_t r = next_static;
      next_static += G;
      if (next_static >= nstatic) claimed = claim();
      return r;
    }
    if (cur < cur_end && cur < ntiles) return cur++;
    if (claimed < 0) claimed = claim();   // no static tiles for this CTA
    cur = claimed;
    cur_end = claimed + chunk;
    if (cur >= ntiles) return -1;
    claimed = claim();
    return cur++;
  };
  auto issue = [&](int st, int64_t t) {
    meta[st][2] = t;
    if (t < 0) {
      mbar_arrive(&full[st]);
      return;
    }
    const int64_t r0 = t * ROWS, r1 = min(nrows, r0 + ROWS);
    const int64_t s = (int64_t)rowptr[r0], e = (int64_t)rowptr[r1];
    const int64_t sc = s & ~(int64_t)(L::CA - 1), ec = (e + L::CA - 1) & ~(int64_t)(L::CA - 1);
    const int64_t sv0 = s & ~(int64_t)(L::VA - 1), ev = (e + L::VA - 1) & ~(int64_t)(L::VA - 1);
    const bool direct = !(tma_ok & 1) || e <= s || e - s > CAP || ec > nnz_end || ev > nnz_end;
    const bool rp_staged = (tma_ok & 2) && r0 + L::RP_N <= nrows + 1;
    meta[st][0] = direct ? -1 : sc;
    meta[st][1] = sv0;
    meta[st][3] = s;
    meta[st][4] = e;
    meta[st][5] = rp_staged;
    const uint32_t bc = direct ? 0 : (uint32_t)((ec - sc) * sizeof(CI));
    const uint32_t bv = direct ? 0 : (uint32_t)((ev - sv0) * sizeof(T));
    const uint32_t br = rp_staged ? (uint32_t)(L::RP_N * sizeof(RP)) : 0;
    if (bc + bv + br == 0) {
      mbar_arrive(&full[st]);
    } else {
      mbar_arrive_expect_tx(&full[st], bc + bv + br);
      if (!direct) {
        bulk_g2s(sci(st), colind + sc, bc, &full[st]);
        bulk_g2s(sv(st), values + sv0, bv, &full[st]);
      }
      if (rp_staged) bulk_g2s(srp(st), rowptr + r0, br, &full[st]);
    }
  };
  if (tid == 0) {
    for (int st = 0; st < ST; ++st) mbar_init(&full[st], 1);
    fence_barrier_init();
    for (int st = 0; st < ST; ++st) issue(st, next_id());
  }
  __syncthreads();
  for (int64_t it = 0;; ++it) {
    const int st = (int)(it % ST);
    mbar_wait(&full[st], (uint32_t)((it / ST) & 1));
    const int64_t t = meta[st][2];
    if (t < 0) break;
    const int64_t row = t * ROWS + gi;
    // the row's range: from the staged rowptr slice (full tiles), else global
    int64_t b = 0, e = 0;
    if (meta[st][5]) {
      b = (int64_t)srp(st)[gi];
      e = (int64_t)srp(st)[gi + 1];
    } else if (row < nrows) {
      b = (int64_t)rowptr[row];
      e = (int64_t)rowptr[row + 1];
    }
    if (e < b) e = b;
    const int64_t sc = meta[st][0], sv0 = meta[st][1];
    const int64_t tile_s = meta[st][3], tile_e = meta[st][4];
    const bool staged = sc >= 0 && b >= tile_s && e <= tile_e;
    T acc;
    if (__all_sync(0xffffffffu, staged || row >= nrows))
      acc = row_fold<T, CI, MC>(sci(st) + (b - sc), sv(st) + (b - sv0), (int)(e - b), x);
    else
      acc = row_fold<T, CI, MC>(colind + b, values + b, (int)(e - b), x);
    if (row < nrows) y[row] = acc;
    __syncthreads();
    if (tid == 0) {
      fence_proxy_async();
      issue(st, next_id());
    }
  }
  if (dbg && tid == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_rs_times[3 * blockIdx.x] = t_start;
    g_rs_times[3 * blockIdx.x + 1] = global_ns();
    g_rs_times[3 * blockIdx.x + 2] = smid;
  }
}

// structure analysis for the plan: longest row, and whether rowptr is monotone
// (stats[1] != 0 when some row has rowptr[r+1] < rowptr[r])
template <class RP>
__global__ void row_stats_kernel(int64_t nrows, const RP* __restrict__ rowptr,
                                 unsigned long long* __restrict__ stats) {
  int64_t local = 0;
  int desc = 0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t len = (int64_t)rowptr[r + 1] - (int64_t)rowptr[r];
    local = len > local ? len : local;
    desc |= len < 0;
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const int64_t o = __shfl_xor_sync(0xffffffffu, local, off);
    local = o > local ? o : local;
  }
  desc = __any_sync(0xffffffffu, desc);
  if ((threadIdx.x & 31) == 0 && local > 0) atomicMax(stats, (unsigned long long)local);
  if ((threadIdx.x & 31) == 0 && desc) atomicOr(stats + 1, 1ull);
}

// ================================================================ host side
struct CsrPlanImpl {
  int64_t nrows = 0, nnz = 0, ntiles = 0;
  int64_t* tile_row = nullptr;  // device, 2 * (ntiles + 1): tile_row then tile_nnz
  int device = 0;
  int64_t max_len = 0;          // longest row
  int exact_vl = 0;             // > 0: regular structure -> vector kernel with this VL
  int exact = 0;                // 1: fp64 / int rows folded in the reference order too
  int warpblock = 0;            // 1: warp-block kernel (irregular monotone structures)
  int rowstream = 0;            // > 0: row-stream kernel for the reference-order fold (staged entries per row)
  int rowstream_all = 0;        // 1: row-stream kernel in tree mode too (LAPIS_B200_SPMV_KERNEL=rs)
};

static int64_t ntiles_for(int64_t nrows, int64_t nnz) {
  const int64_t total = nrows + nnz;
  return (total + TILE_KEYS - 1) / TILE_KEYS;
}

int launch_partition(int64_t nrows, const void* rowptr, int rp_bytes, int64_t ntiles,
                     int64_t* tile_row, cudaStream_t st, RowGuard guard = RowGuard()) {
  const int threads = 256;
  const int64_t blocks = (nrows + 1 + threads - 1) / threads;
  int64_t* tile_nnz = tile_row + (ntiles + 1);
  if (rp_bytes == 8)
    tile_partition_kernel<int64_t><<<(unsigned)blocks, threads, 0, st>>>(
        nrows, (const int64_t*)rowptr, ntiles, tile_row, tile_nnz, guard);
  else
    tile_partition_kernel<int32_t><<<(unsigned)blocks, threads, 0, st>>>(
        nrows, (const int32_t*)rowptr, ntiles, tile_row, tile_nnz, guard);
  return check_launch("tile_partition_kernel");
}

template <class T, class RP, class CI, int NT, int ST>
static int launch_tile_cfg(int64_t ntiles, const void* rowptr, const void* colind,
                           const void* values, const void* x, void* y, const int64_t* tile_row,
                           cudaStream_t st, RowGuard guard) {
  using L = StreamSmem<T, CI, ST>;
  auto kern = spmv_tile_kernel<T, RP, CI, NT, ST>;
  static thread_local int configured_dev = -1;
  static thread_local int ctas_per_sm = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    LB_TRY(check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)L::TOTAL), "smem attr (spmv_tile_kernel)"));
    LB_TRY(check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas_per_sm, kern, NT,
                                                                    L::TOTAL), "occupancy"));
    if (ctas_per_sm < 1) ctas_per_sm = 1;
    configured_dev = dev;
  }
  const int tma_ok = ((uintptr_t)colind % 16 == 0) && ((uintptr_t)values % 16 == 0);
  int64_t grid = (int64_t)num_sms() * ctas_per_sm;
  if (grid > ntiles) grid = ntiles;
  if (grid < 1) grid = 1;
  const int64_t* tile_nnz = tile_row + (ntiles + 1);
  kern<<<(unsigned)grid, NT, L::TOTAL, st>>>((const RP*)rowptr, (const CI*)colind,
                                             (const T*)values, (const T*)x, (T*)y, tile_row,
                                             tile_nnz, ntiles, tma_ok, guard);
  return check_launch("spmv_tile_kernel");
}

// kernel shape (threads per CTA, ring depth); LAPIS_B200_SPMV_CFG selects a
// variant for tuning runs (0 = default)
static int spmv_cfg() {
  static int cfg = [] {
    const char* e = getenv("LAPIS_B200_SPMV_CFG");
    return e ? atoi(e) : 0;
  }();
  return cfg;
}

template <class T, class RP, class CI>
static int launch_tile_t(int64_t ntiles, const void* rowptr, const void* colind,
                         const void* values, const void* x, void* y, const int64_t* tile_row,
                         cudaStream_t st, RowGuard g = RowGuard()) {
  switch (spmv_cfg()) {
    case 1: return launch_tile_cfg<T, RP, CI, 128, 4>(ntiles, rowptr, colind, values, x, y, tile_row, st, g);
    case 2: return launch_tile_cfg<T, RP, CI, 256, 3>(ntiles, rowptr, colind, values, x, y, tile_row, st, g);
    case 3: return launch_tile_cfg<T, RP, CI, 128, 3>(ntiles, rowptr, colind, values, x, y, tile_row, st, g);
    default: return launch_tile_cfg<T, RP, CI, 256, 4>(ntiles, rowptr, colind, values, x, y, tile_row, st, g);
  }
}

template <class T, class RP, class CI, int NT, int PER, int ST, int MC>
static int launch_rowstream_cfg(int64_t nrows, const void* rowptr, const void* colind,
                                const void* values, const void* x, void* y, cudaStream_t st,
                                RowGuard guard) {
  constexpr int ROWS = NT, CAP = ROWS * PER;
  using L = RowStreamSmem<T, CI, RP, NT, CAP, ST>;
  auto kern = spmv_rowstream_kernel<T, RP, CI, NT, CAP, ST, MC>;
  static int configured[64] = {0};
  static int ctas_per_sm[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!configured[dev]) {
    LB_TRY(check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)L::TOTAL), "smem attr (spmv_rowstream_kernel)"));
    int c = 0;
    LB_TRY(check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, kern, NT, L::TOTAL),
                      "occupancy"));
    ctas_per_sm[dev] = c < 1 ? 1 : c;
    configured[dev] = 1;
  }
  // bit 0: entry arrays 16-byte aligned (bulk copies of colind / values);
  // bit 1: rowptr too (bulk copies of each tile's row offsets)
  const int tma_ok = (((uintptr_t)colind % 16 == 0) && ((uintptr_t)values % 16 == 0)) |
                     (((uintptr_t)rowptr % 16 == 0) ? 2 : 0);
  const int64_t ntiles = (nrows + ROWS - 1) / ROWS;
  int64_t grid = (int64_t)num_sms() * ctas_per_sm[dev];
  if (grid > ntiles) grid = ntiles;
  if (grid < 1) grid = 1;
  // tile split: the first (100 - LAPIS_B200_RS_DYN) % of the tiles static
  // (CTA b takes b, b + G, ...), the rest from a counter in runs of
  // LAPIS_B200_RS_CHUNK consecutive tiles per atomic (default: all tiles,
  // runs of 5; problems of at least 16 tiles per CTA unless the variable is
  // set).  C5, per launch (scripts/c5_dyn.sh, c5_chunk.sh): all static
  // 11.9-12.2 ms with straggler launches at 12.7-14.2 (a few CTAs end 1.2-2.4
  // ms after the rest); all counter, one tile per atomic 14.8 ms (the single
  // counter's contention); runs of 2 / 3 / 4 / 5 / 6 / 7 / 10 / 12 / 16 tiles
  // 12.3 / 12.54 / 12.05 / 11.80 / 11.87 / 11.96 / 11.87 / 12.18 / 12.47 ms,
  // every CTA ending within 0.02 ms
  const char* dyn_env = getenv("LAPIS_B200_RS_DYN");
  const int dyn_pct = dyn_env ? std::max(0, std::min(100, atoi(dyn_env))) : 100;
  const char* chunk_env = getenv("LAPIS_B200_RS_CHUNK");
  const int chunk = chunk_env ? std::max(1, atoi(chunk_env)) : 5;
  int64_t nstatic = ntiles;
  unsigned long long* next_tile = nullptr;
  if (dyn_pct > 0 && (dyn_env != nullptr || ntiles >= 16 * grid)) {
    nstatic = ntiles - ntiles * dyn_pct / 100;
    LB_TRY(check_cuda(cudaMallocAsync((void**)&next_tile, sizeof(*next_tile), st),
                      "alloc(row-stream counter)"));
    LB_TRY(check_cuda(cudaMemsetAsync(next_tile, 0, sizeof(*next_tile), st), "memset(counter)"));
  }
  static const char* times_path = getenv("LAPIS_B200_RS_TIMES");
  if (times_path) {
    const int one = 1;
    cudaMemcpyToSymbolAsync(g_rs_dbg, &one, sizeof(int), 0, cudaMemcpyHostToDevice, st);
  }
  kern<<<(unsigned)grid, NT, L::TOTAL, st>>>(nrows, (const RP*)rowptr, (const CI*)colind,
                                             (const T*)values, (const T*)x, (T*)y, tma_ok, nstatic,
                                             next_tile, chunk, guard);
  if (next_tile) cudaFreeAsync(next_tile, st);
  if (times_path) {
    static unsigned long long h[3 * 4096];
    const int n = (int)std::min<int64_t>(grid, 4096);
    cudaMemcpyFromSymbolAsync(h, g_rs_times, sizeof(unsigned long long) * 3 * n, 0,
                              cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if (FILE* f = fopen(times_path, "a")) {
      fprintf(f, "launch %d %lld\n", n, (long long)ntiles);
      for (int i = 0; i < n; ++i) fprintf(f, "%llu %llu %llu\n", h[3 * i], h[3 * i + 1], h[3 * i + 2]);
      fclose(f);
    }
  }
  return check_launch("spmv_rowstream_kernel");
}

// staged entries per row class of the row-stream kernel; 0 = not used
// (rows of <= 14 entries stay on the exact vector kernel: C1's 5-point rows
// measured 20 us there against 20-88 us for row-stream shapes)
static int rowstream_per(double mean) {
  if (mean > 14.0 && mean <= 28.0) return 32;
  return 0;
}
// LAPIS_B200_RS_CFG selects a shape variant for tuning runs (0 = default)
static int rowstream_cfg() {
  static int cfg = [] {
    const char* e = getenv("LAPIS_B200_RS_CFG");
    return e ? atoi(e) : 0;
  }();
  return cfg;
}

template <class T, class RP, class CI>
struct RowStreamOp {
  static int run(int per, int64_t nrows, const void* rp, const void* ci, const void* v,
                 const void* x, void* y, cudaStream_t st, RowGuard g) {
    // (NT threads = rows per tile, PER staged entries per row, ST stages, MC).
    // Measured on a 24M-row 27-point stencil (exact): NT = 64, 2 stages
    // (five CTAs per SM) 5.77 TB/s; NT = 96 5.53; NT = 128 5.09; NT = 256
    // 4.92; NT = 32 5.2; NT = 64 with 3 stages 3.6, with MC = 8 5.24 (the
    // vector kernel: tree 5.59, exact 4.72).  Full config 5 (200M rows):
    // 5.14 TB/s exact vs 4.37 for the exact vector kernel.
    switch (rowstream_cfg()) {
      case 1: return launch_rowstream_cfg<T, RP, CI, 32, 28, 2, 16>(nrows, rp, ci, v, x, y, st, g);
      case 2: return launch_rowstream_cfg<T, RP, CI, 128, 28, 2, 16>(nrows, rp, ci, v, x, y, st, g);
      default: break;
    }
    (void)per;
    return launch_rowstream_cfg<T, RP, CI, 64, 28, 2, 16>(nrows, rp, ci, v, x, y, st, g);
  }
};

template <class T, class RP, class CI, int VL, bool EXACT>
static int launch_vector_t(int64_t nrows, const void* rowptr, const void* colind,
                           const void* values, const void* x, void* y, cudaStream_t st,
                           RowGuard guard = RowGuard()) {
  const int threads = 256;
  int64_t blocks = (nrows * VL + threads - 1) / threads;
  // grid cap in CTAs per SM (LAPIS_B200_SPMV_BLOCKS_PER_SM for tuning runs).
  // Measured on C5 (200M rows, VL = 4): 8 / 64 / 256 / 1024 / 4096 / uncapped
  // -> 13.9 / 12.8 / 12.0 / 11.9 / 12.2 / 13.3 ms: many short-lived CTAs
  // balance better than a few long grid-stride walkers, and neighbouring CTAs
  // stream neighbouring rows (x reuse in L2)
  // Small problems (at most 8 waves of 8 CTAs per SM) run as one resident
  // wave walking the rows grid-stride: C1 (1M rows, VL = 1) 20.5 -> 19.5 us
  // per step (4 CTAs per SM: 23.3, 16: 20.3)
  static const int64_t per_sm_env = [] {
    const char* e = getenv("LAPIS_B200_SPMV_BLOCKS_PER_SM");
    return (int64_t)(e ? atoi(e) : 0);
  }();
  const int64_t wave = (int64_t)num_sms() * 8;
  // the no-plan call's guarded launch for decreasing rowptrs (rare; skipped
  // otherwise) walks the rows from 64 CTAs per SM: a 1024-per-SM grid costs
  // ~0.16 ms of CTA launches even when every CTA exits at the guard (C5)
  const bool rare = guard.stats != nullptr && guard.want == 3;
  const int64_t per_sm = per_sm_env > 0 ? per_sm_env
                                        : (blocks <= 8 * wave ? 8 : (rare ? 64 : 1024));
  const int64_t cap = (int64_t)num_sms() * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  // one-wave problems (C1: ~15 us of kernel behind ~2 us of launch): launched
  // with programmatic stream serialization, so the grid is set up while the
  // previous one drains (LAPIS_B200_PDL=0: plain launch)
  static const bool pdl = [] {
    const char* e = getenv("LAPIS_B200_PDL");
    return !(e && e[0] == '0');
  }();
  if (pdl && per_sm_env == 0 && blocks <= wave) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    LB_TRY(check_cuda(cudaLaunchKernelEx(&cfg, spmv_vector_kernel<T, RP, CI, VL, EXACT>, nrows,
                                         (const RP*)rowptr, (const CI*)colind, (const T*)values,
                                         (const T*)x, (T*)y, guard),
                      "launch spmv_vector_kernel (PDL)"));
    return check_launch("spmv_vector_kernel");
  }
  spmv_vector_kernel<T, RP, CI, VL, EXACT><<<(unsigned)blocks, threads, 0, st>>>(
      nrows, (const RP*)rowptr, (const CI*)colind, (const T*)values, (const T*)x, (T*)y, guard);
  return check_launch("spmv_vector_kernel");
}

template <class T, class RP, class CI>
static int launch_warpblock_t(int64_t nrows, const void* rowptr, const void* colind,
                              const void* values, const void* x, void* y, int exact,
                              unsigned long long* next, cudaStream_t st, RowGuard guard) {
  static const bool pol = [] {
    const char* e = getenv("LAPIS_B200_SPMV_WB_POLICY");  // A/B runs: 0 = plain loads
    return !(e && e[0] == '0');
  }();
  static const int wbu = [] {
    const char* e = getenv("LAPIS_B200_SPMV_WB_U");  // A/B runs: entries per lane per window
    return e ? atoi(e) : 16;
  }();
  auto kern = exact ? (pol ? spmv_warpblock_kernel<T, RP, CI, 8, true, true>
                           : spmv_warpblock_kernel<T, RP, CI, 8, true, false>)
                    : (pol ? spmv_warpblock_kernel<T, RP, CI, 8, false, true>
                           : spmv_warpblock_kernel<T, RP, CI, 8, false, false>);
  if (wbu == 16 && pol)
    kern = exact ? spmv_warpblock_kernel<T, RP, CI, 16, true, true>
                 : spmv_warpblock_kernel<T, RP, CI, 16, false, true>;
  if (wbu == 24 && pol)
    kern = exact ? spmv_warpblock_kernel<T, RP, CI, 24, true, true>
                 : spmv_warpblock_kernel<T, RP, CI, 24, false, true>;
  static thread_local int configured_dev = -1;
  static thread_local int ctas_per_sm[2] = {0, 0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {  // one resident wave of the persistent grid
    for (int ex = 0; ex < 2; ++ex) {
      auto kk = ex ? spmv_warpblock_kernel<T, RP, CI, 8, true> : spmv_warpblock_kernel<T, RP, CI, 8, false>;
      LB_TRY(check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas_per_sm[ex], kk, 256, 0),
                        "occupancy"));
      if (ctas_per_sm[ex] < 1) ctas_per_sm[ex] = 1;
    }
    configured_dev = dev;
  }
  const int64_t nblk = (nrows + 31) / 32;
  int64_t blocks = (nblk + 7) / 8;
  const int64_t cap = (int64_t)num_sms() * ctas_per_sm[exact ? 1 : 0];
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  if (next) LB_TRY(check_cuda(cudaMemsetAsync(next, 0, sizeof(*next), st), "memset(spmv counter)"));
  kern<<<(unsigned)blocks, 256, 0, st>>>(nrows, (const RP*)rowptr, (const CI*)colind,
                                         (const T*)values, (const T*)x, (T*)y, next, guard);
  return check_launch("spmv_warpblock_kernel");
}

template <class T, class RP, class CI, bool EXACT>
static int dispatch_vl(int vl, int64_t nrows, const void* rowptr, const void* colind,
                       const void* values, const void* x, void* y, cudaStream_t st,
                       RowGuard g = RowGuard()) {
  switch (vl) {
    case 1: return launch_vector_t<T, RP, CI, 1, EXACT>(nrows, rowptr, colind, values, x, y, st, g);
    case 2: return launch_vector_t<T, RP, CI, 2, EXACT>(nrows, rowptr, colind, values, x, y, st, g);
    case 4: return launch_vector_t<T, RP, CI, 4, EXACT>(nrows, rowptr, colind, values, x, y, st, g);
    case 8: return launch_vector_t<T, RP, CI, 8, EXACT>(nrows, rowptr, colind, values, x, y, st, g);
    case 16: return launch_vector_t<T, RP, CI, 16, EXACT>(nrows, rowptr, colind, values, x, y, st, g);
    case 32: return launch_vector_t<T, RP, CI, 32, EXACT>(nrows, rowptr, colind, values, x, y, st, g);
  }
  return fail(LAPIS_B200_ERR_ARG, "spmv: vector_length must be 0 or a power of two <= 32");
}

// type dispatch: F(T, RP, CI)
template <template <class, class, class> class F, class... Args>
static int dispatch_types(int dtype, int rp_bytes, int ci_bytes, Args&&... args) {
#define LB_CI(T, RP)                                                        \
  return ci_bytes == 8 ? F<T, RP, int64_t>::run(std::forward<Args>(args)...) \
                       : F<T, RP, int32_t>::run(std::forward<Args>(args)...)
#define LB_RP(T) \
  if (rp_bytes == 8) { LB_CI(T, int64_t); } else { LB_CI(T, int32_t); }
  switch (dtype) {
    case LAPIS_B200_F64: LB_RP(double)
    case LAPIS_B200_F32: LB_RP(float)
    case LAPIS_B200_I64: LB_RP(long long)
    case LAPIS_B200_I32: LB_RP(int)
  }
#undef LB_RP
#undef LB_CI
  return fail(LAPIS_B200_ERR_ARG, "unsupported dtype");
}

template <class T, class RP, class CI>
struct TileOp {
  static int run(int64_t ntiles, const void* rp, const void* ci, const void* v,
                 const void* x, void* y, const int64_t* tr, cudaStream_t st,
                 RowGuard g = RowGuard()) {
    return launch_tile_t<T, RP, CI>(ntiles, rp, ci, v, x, y, tr, st, g);
  }
};
template <class T, class RP, class CI>
struct VecExactGuardedOp {
  static int run(int vl, int64_t nrows, const void* rp, const void* ci, const void* v,
                 const void* x, void* y, cudaStream_t st, RowGuard g) {
    return dispatch_vl<T, RP, CI, true>(vl, nrows, rp, ci, v, x, y, st, g);
  }
};
template <class T, class RP, class CI>
struct VecOp {
  static int run(int vl, int64_t nrows, const void* rp, const void* ci, const void* v,
                 const void* x, void* y, cudaStream_t st) {
    return dispatch_vl<T, RP, CI, false>(vl, nrows, rp, ci, v, x, y, st);
  }
};
template <class T, class RP, class CI>
struct WarpBlockOp {
  static int run(int64_t nrows, const void* rp, const void* ci, const void* v, const void* x,
                 void* y, int exact, cudaStream_t st, RowGuard g = RowGuard()) {
    // the block counter: a per-call stream-ordered allocation (pool-cached),
    // so multiplies with one plan on several streams never share it
    unsigned long long* next = nullptr;
    LB_TRY(check_cuda(cudaMallocAsync((void**)&next, sizeof(*next), st), "alloc(spmv counter)"));
    const int rc = launch_warpblock_t<T, RP, CI>(nrows, rp, ci, v, x, y, exact, next, st, g);
    cudaFreeAsync(next, st);
    return rc;
  }
};
template <class T, class RP, class CI>
struct VecExactOp {
  static int run(int vl, int64_t nrows, const void* rp, const void* ci, const void* v,
                 const void* x, void* y, cudaStream_t st) {
    return dispatch_vl<T, RP, CI, true>(vl, nrows, rp, ci, v, x, y, st);
  }
};

static int validate(int64_t nrows, int64_t ncols, int64_t nnz, const void* rowptr, int rp_bytes,
                    const void* colind, int ci_bytes, const void* values, const void* x,
                    const void* y, int dtype) {
  if (nrows < 0 || ncols < 0 || nnz < 0) return fail(LAPIS_B200_ERR_ARG, "spmv: negative extent");
  if (!valid_dtype(dtype)) return fail(LAPIS_B200_ERR_ARG, "spmv: unsupported dtype");
  if ((rp_bytes != 4 && rp_bytes != 8) || (ci_bytes != 4 && ci_bytes != 8))
    return fail(LAPIS_B200_ERR_ARG, "spmv: index widths must be 4 or 8 bytes");
  if (!rowptr) return fail(LAPIS_B200_ERR_ARG, "spmv: null rowptr");
  if (nrows > 0 && !y) return fail(LAPIS_B200_ERR_ARG, "spmv: null y");
  if (nnz > 0 && (!colind || !values || !x)) return fail(LAPIS_B200_ERR_ARG, "spmv: null operand");
  if (rp_bytes == 4 && nnz > 0x7fffffffLL)
    return fail(LAPIS_B200_ERR_ARG, "spmv: nnz exceeds an i32 rowptr");
  return LAPIS_B200_OK;
}

int spmv_csr(int64_t nrows, int64_t ncols, int64_t nnz, const void* rowptr, int rp_bytes,
             const void* colind, int ci_bytes, const void* values, const void* x, void* y,
             int dtype, int vl, cudaStream_t st) {
  LB_TRY(validate(nrows, ncols, nnz, rowptr, rp_bytes, colind, ci_bytes, values, x, y, dtype));
  if (nrows == 0) return LAPIS_B200_OK;
  if (vl != 0) return dispatch_types<VecOp>(dtype, rp_bytes, ci_bytes, vl, nrows, rowptr, colind,
                                            values, x, y, st);
  // no plan: one stats pass over rowptr on the device, then the candidate
  // kernels launched behind a device guard — the exact vector kernel (the
  // plan's choice for regular structures, bit-identical), the warp-block
  // kernel (monotone irregular) or, for a rowptr that decreases somewhere,
  // the exact one-row-per-lane vector kernel, which clamps each row to
  // range(begin, max(begin, end)) (interp.py:808) — so the call stays
  // asynchronous.  (The tile kernel's key-balanced partition assumes a
  // non-decreasing rowptr, so it is never chosen for such structures.)
  unsigned long long* stats = nullptr;
  LB_TRY(check_cuda(cudaMallocAsync((void**)&stats, 2 * sizeof(unsigned long long), st),
                    "cudaMallocAsync(spmv stats)"));
  int rc = check_cuda(cudaMemsetAsync(stats, 0, 2 * sizeof(unsigned long long), st), "memset(stats)");
  if (rc == LAPIS_B200_OK) {
    const int64_t blocks = std::min<int64_t>((nrows + 255) / 256, (int64_t)num_sms() * 8);
    if (rp_bytes == 8)
      row_stats_kernel<int64_t><<<(unsigned)blocks, 256, 0, st>>>(nrows, (const int64_t*)rowptr, stats);
    else
      row_stats_kernel<int32_t><<<(unsigned)blocks, 256, 0, st>>>(nrows, (const int32_t*)rowptr, stats);
    rc = check_launch("row_stats_kernel");
  }
  const double mean = (double)nnz / (double)nrows;
  int cvl = 1;
  while (cvl < 8 && (double)(cvl * 2) * 6.0 <= mean) cvl *= 2;
  RowGuard greg, gwb, girr;
  greg.stats = gwb.stats = girr.stats = stats;
  greg.thresh = gwb.thresh = girr.thresh = (long long)std::max(64.0, 8.0 * mean);  // analyse_rows
  greg.want = 1;  // regular: exact vector kernel
  gwb.want = 2;   // monotone irregular: warp-block kernel (the plan's choice)
  girr.want = 3;  // decreasing rowptr: exact vector kernel, one row per lane
  // regular: the row-stream kernel (reference order, structure streamed by the
  // TMA engine) when the mean row fits its stage, else the exact vector kernel
  const int per = rowstream_per(mean);
  if (rc == LAPIS_B200_OK && per > 0)
    rc = dispatch_types<RowStreamOp>(dtype, rp_bytes, ci_bytes, per, nrows, rowptr, colind, values,
                                     x, y, st, greg);
  else if (rc == LAPIS_B200_OK)
    rc = dispatch_types<VecExactGuardedOp>(dtype, rp_bytes, ci_bytes, cvl, nrows, rowptr, colind,
                                           values, x, y, st, greg);
  if (rc == LAPIS_B200_OK)
    rc = dispatch_types<WarpBlockOp>(dtype, rp_bytes, ci_bytes, nrows, rowptr, colind, values, x,
                                     y, dtype == LAPIS_B200_F32 ? 1 : 0, st, gwb);
  if (rc == LAPIS_B200_OK)
    rc = dispatch_types<VecExactGuardedOp>(dtype, rp_bytes, ci_bytes, 1, nrows, rowptr, colind,
                                           values, x, y, st, girr);
  cudaFreeAsync(stats, st);
  return rc;
}

// Regular structures (longest row within 8x the mean, or <= 64) take the exact
// vector kernel with VL = pow2floor(mean / 6) in [1, 8]; anything else the
// key-balanced tile kernel.  One device->host read at plan creation.
static int analyse_rows(CsrPlanImpl* p, const void* rowptr, int rp_bytes, cudaStream_t st) {
  unsigned long long* d = nullptr;
  LB_TRY(check_cuda(cudaMallocAsync((void**)&d, 2 * sizeof(unsigned long long), st), "alloc(stats)"));
  int rc = check_cuda(cudaMemsetAsync(d, 0, 2 * sizeof(unsigned long long), st), "memset(stats)");
  if (rc == LAPIS_B200_OK) {
    const int64_t blocks = std::min<int64_t>((p->nrows + 255) / 256, (int64_t)num_sms() * 8);
    if (rp_bytes == 8)
      row_stats_kernel<int64_t><<<(unsigned)blocks, 256, 0, st>>>(p->nrows, (const int64_t*)rowptr, d);
    else
      row_stats_kernel<int32_t><<<(unsigned)blocks, 256, 0, st>>>(p->nrows, (const int32_t*)rowptr, d);
    rc = check_launch("row_stats_kernel");
  }
  unsigned long long h[2] = {0, 0};
  if (rc == LAPIS_B200_OK)
    rc = check_cuda(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, st), "stats D2H");
  if (rc == LAPIS_B200_OK) rc = check_cuda(cudaStreamSynchronize(st), "stats sync");
  cudaFreeAsync(d, st);
  if (rc != LAPIS_B200_OK) return rc;
  p->max_len = (int64_t)h[0];
  const bool monotone = h[1] == 0;
  const double mean = p->nrows > 0 ? (double)p->nnz / (double)p->nrows : 0.0;
  int vl = 1;
  while (vl < 8 && (double)(vl * 2) * 6.0 <= mean) vl *= 2;
  const char* force = getenv("LAPIS_B200_SPMV_VL");
  if (force) vl = atoi(force);
  const bool regular = p->max_len <= 64 || (double)p->max_len <= 8.0 * mean;
  p->exact_vl = (force && vl > 0) ? vl : (regular ? vl : 0);
  // a decreasing rowptr: the exact vector kernel with one row per lane (it
  // clamps every row to range(begin, max(begin, end)), interp.py:808); the
  // tile partition and the warp-block entry runs assume a monotone rowptr
  if (!monotone) p->exact_vl = 1;
  const char* ex = getenv("LAPIS_B200_SPMV_EXACT");
  p->exact = (ex && atoi(ex) != 0) ? 1 : 0;
  // warp-block kernel: irregular monotone structures (power-law rows: 1.46 vs
  // 1.73 ms for the tile kernel on config 3's matrix, before the dynamic
  // blocks and the cooperative hub-row fold); LAPIS_B200_SPMV_KERNEL = wb /
  // vec / tile forces a choice for tuning runs
  const char* kf = getenv("LAPIS_B200_SPMV_KERNEL");
  bool wb = monotone && !force && (!regular || mean < WARPBLOCK_MAX_MEAN);
  if (kf && !strcmp(kf, "wb")) wb = monotone;
  if (kf && (!strcmp(kf, "vec") || !strcmp(kf, "tile") || !strcmp(kf, "rs"))) wb = false;
  p->warpblock = wb ? 1 : 0;
  // row-stream kernel: the reference-order fold of regular monotone structures
  // (C1, C5 exact, fp32); LAPIS_B200_SPMV_KERNEL = vec keeps the vector kernel
  const bool vec_forced = kf && !strcmp(kf, "vec");
  p->rowstream = (monotone && regular && !wb && !vec_forced && !force) ? rowstream_per(mean) : 0;
  if (kf && !strcmp(kf, "rs") && monotone) p->rowstream = rowstream_per(mean) ? rowstream_per(mean) : 32;
  // ... in tree mode too: the sequential row sum is within the tree mode's
  // tolerance and, with the counter-scheduled tiles, the faster kernel (C5
  // 11.82 vs 12.13-12.16 ms back to back for the VL = 4 tree, which also
  // runs into the power cap); LAPIS_B200_RS_TREE=0 keeps the vector kernel
  const char* rt = getenv("LAPIS_B200_RS_TREE");
  p->rowstream_all = ((kf && !strcmp(kf, "rs")) || (p->rowstream > 0 && !(rt && atoi(rt) == 0))) ? 1 : 0;
  return LAPIS_B200_OK;
}

int csr_plan_create(int64_t nrows, int64_t nnz, const void* rowptr, int rp_bytes,
                    cudaStream_t st, void** out) {
  if (!out) return fail(LAPIS_B200_ERR_ARG, "plan: null out pointer");
  *out = nullptr;
  if (nrows < 0 || nnz < 0 || !rowptr || (rp_bytes != 4 && rp_bytes != 8))
    return fail(LAPIS_B200_ERR_ARG, "plan: bad arguments");
  auto* p = new CsrPlanImpl();
  p->nrows = nrows;
  p->nnz = nnz;
  p->ntiles = ntiles_for(nrows, nnz);
  cudaGetDevice(&p->device);
  int rc = check_cuda(cudaMalloc((void**)&p->tile_row, 2 * (p->ntiles + 1) * sizeof(int64_t)),
                      "cudaMalloc(plan)");

  if (rc == LAPIS_B200_OK && nrows > 0)
    rc = launch_partition(nrows, rowptr, rp_bytes, p->ntiles, p->tile_row, st);
  if (rc == LAPIS_B200_OK && nrows > 0) rc = analyse_rows(p, rowptr, rp_bytes, st);
  if (rc != LAPIS_B200_OK) {
    if (p->tile_row) cudaFree(p->tile_row);
    delete p;
    return rc;
  }
  *out = p;
  return LAPIS_B200_OK;
}

int csr_plan_info(void* plan, int64_t* out4) {
  auto* p = static_cast<CsrPlanImpl*>(plan);
  if (!p || !out4) return fail(LAPIS_B200_ERR_ARG, "plan_info: null argument");
  out4[0] = p->max_len;
  out4[1] = p->exact_vl;
  out4[2] = p->ntiles;
  out4[3] = p->exact | (p->warpblock << 1) | ((p->rowstream > 0) << 2) | (p->rowstream_all << 3);
  return LAPIS_B200_OK;
}

int csr_plan_set_exact(void* plan, int exact) {
  auto* p = static_cast<CsrPlanImpl*>(plan);
  if (!p) return fail(LAPIS_B200_ERR_ARG, "plan_set_exact: null plan");
  p->exact = exact ? 1 : 0;
  return LAPIS_B200_OK;
}

int csr_plan_destroy(void* plan) {
  auto* p = static_cast<CsrPlanImpl*>(plan);
  if (!p) return LAPIS_B200_OK;
  int rc = check_cuda(cudaFree(p->tile_row), "cudaFree(plan)");
  delete p;
  return rc;
}

int spmv_csr_plan(void* plan, const void* rowptr, int rp_bytes, const void* colind, int ci_bytes,
                  const void* values, const void* x, void* y, int dtype, cudaStream_t st) {
  auto* p = static_cast<CsrPlanImpl*>(plan);
  if (!p) return fail(LAPIS_B200_ERR_ARG, "spmv: null plan");
  LB_TRY(validate(p->nrows, 0, p->nnz, rowptr, rp_bytes, colind, ci_bytes, values, x, y, dtype));
  if (p->nrows == 0) return LAPIS_B200_OK;
  if (p->warpblock)  // rows <= LONG_ROW in order; longer: warp tree unless exact / fp32
    return dispatch_types<WarpBlockOp>(dtype, rp_bytes, ci_bytes, p->nrows, rowptr, colind,
                                       values, x, y,
                                       (p->exact || dtype == LAPIS_B200_F32) ? 1 : 0, st);
  const bool ordered = p->exact || dtype == LAPIS_B200_F32 || p->exact_vl == 1;
  if (p->rowstream > 0 && (ordered || p->rowstream_all))
    return dispatch_types<RowStreamOp>(dtype, rp_bytes, ci_bytes, p->rowstream, p->nrows, rowptr,
                                       colind, values, x, y, st, RowGuard());
  if (p->exact_vl > 0) {
    // fp32 always folds in the reference order (its 1e-5 contract cannot absorb
    // reassociation on long rows); fp64 / ints take the emitted-mapping tree
    // (ThreadVectorRange reduce) unless exact mode was requested
    // (VL = 1: both are the sequential row sum; the exact kernel's two-entry
    // unroll keeps more loads in flight — C1 21.5 vs 26 us measured)
    if (ordered)
      return dispatch_types<VecExactOp>(dtype, rp_bytes, ci_bytes, p->exact_vl, p->nrows, rowptr,
                                        colind, values, x, y, st);
    return dispatch_types<VecOp>(dtype, rp_bytes, ci_bytes, p->exact_vl, p->nrows, rowptr,
                                 colind, values, x, y, st);
  }
  return dispatch_types<TileOp>(dtype, rp_bytes, ci_bytes, p->ntiles, rowptr, colind, values, x,
                                y, (const int64_t*)p->tile_row, st);
}

}  // namespace lapis_b200
