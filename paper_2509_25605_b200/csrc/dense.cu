// dense.cu — reference-order dense kernels for sm_100a:
//   * gemm_exact / batch_gemm_exact: C[i,j] = sum_k A[i,k]*B[k,j] with the
//     k loop ascending and non-contracted mul/add per step — the order of
//     interp.py:711-722 / 746-763 and of the emitted TeamPolicy nest
//     (golden/cpp/matmul_f64.hpp:23-38), hence bit-identical for every dtype
//     (ints wrap).  Shared-memory tiled so A and B are read once per tile.
//   * gemv: one thread per row (RangePolicy(0, m) of runtime_header.py:268-282)
//     summing sequentially, with A staged through shared memory in 32-column
//     slabs so the HBM reads stay coalesced although each thread walks a row.
//   * reduce_2d: the parallel_reduce family (interp.py:779-795) with the
//     reference combiners and identities; same staging for the row fold.
//   * relu: the GCN elementwise select (cmpf ogt + select).
// The tensor-core fp32 (3xTF32, tcgen05) and fp64 (DMMA) GEMMs live in
// gemm_tf32x3.cu and gemm_dmma.cu.
#include "common.cuh"

#include <algorithm>

#include <cstdlib>

#include <type_traits>

#include <cfloat>
#include <climits>
#include <cmath>

namespace lapis_b200 {

// --------------------------------------------------------------- combiners
template <class T> __device__ __forceinline__ T ident_min();
template <class T> __device__ __forceinline__ T ident_max();
template <> __device__ __forceinline__ double ident_min<double>() { return INFINITY; }
template <> __device__ __forceinline__ double ident_max<double>() { return -INFINITY; }
template <> __device__ __forceinline__ float ident_min<float>() { return INFINITY; }
template <> __device__ __forceinline__ float ident_max<float>() { return -INFINITY; }
template <> __device__ __forceinline__ long long ident_min<long long>() { return LLONG_MAX; }
template <> __device__ __forceinline__ long long ident_max<long long>() { return LLONG_MIN; }
template <> __device__ __forceinline__ int ident_min<int>() { return INT_MAX; }
template <> __device__ __forceinline__ int ident_max<int>() { return INT_MIN; }

template <class T>
__device__ __forceinline__ T identity(int comb) {
  switch (comb) {
    case LAPIS_B200_ADD: return Arith<T>::zero();
    case LAPIS_B200_MUL: return T(1);
    case LAPIS_B200_MIN: return ident_min<T>();
    default: return ident_max<T>();
  }
}

// interp.py:174-183: add/mul rounded; min/max keep acc unless the contribution wins
template <class T>
__device__ __forceinline__ T combine(T acc, T v, int comb) {
  switch (comb) {
    case LAPIS_B200_ADD: return Arith<T>::add(acc, v);
    case LAPIS_B200_MUL: return Arith<T>::mul(acc, v);
    case LAPIS_B200_MIN: return (acc <= v) ? acc : v;
    default: return (acc >= v) ? acc : v;
  }
}

// -------------------------------------------------------------- exact GEMM
constexpr int EG_TILE = 32;   // C tile 32 x 32, K slab 32
constexpr int EG_ROWS = 4;    // outputs per thread (rows)

template <class T, bool RELU>
__global__ void __launch_bounds__(256)
gemm_exact_kernel(int64_t m, int64_t n, int64_t k, const T* __restrict__ A, int64_t lda,
                  const T* __restrict__ B, int64_t ldb, T* __restrict__ C, int64_t ldc,
                  int64_t strideA, int64_t strideB, int64_t strideC, int64_t batch, Guard guard) {
  if (guard_skip(guard)) return;   // fallback launches run only when flagged
  __shared__ T As[EG_TILE][EG_TILE + 1];
  __shared__ T Bs[EG_TILE][EG_TILE + 1];
  // a bounded grid walks the (column, row, batch) tiles, so a guarded launch
  // that does not run costs one wave of CTAs
  const int64_t tn = (n + EG_TILE - 1) / EG_TILE, tm = (m + EG_TILE - 1) / EG_TILE;
  for (int64_t t = blockIdx.x; t < tn * tm * batch; t += gridDim.x) {
  const int64_t bz = t / (tn * tm), by = (t / tn) % tm, bx = t % tn;
  const T* __restrict__ Ab = A + bz * strideA;
  const T* __restrict__ Bb = B + bz * strideB;
  T* __restrict__ Cb = C + bz * strideC;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const int64_t row0 = by * EG_TILE, col0 = bx * EG_TILE;
  T acc[EG_ROWS];
#pragma unroll
  for (int q = 0; q < EG_ROWS; ++q) acc[q] = Arith<T>::zero();
  for (int64_t k0 = 0; k0 < k; k0 += EG_TILE) {
#pragma unroll
    for (int q = 0; q < EG_ROWS; ++q) {
      const int r = ty * EG_ROWS + q;
      const int64_t ar = row0 + r, ak = k0 + tx;
      As[r][tx] = (ar < m && ak < k) ? Ab[ar * lda + ak] : Arith<T>::zero();
      const int64_t bk = k0 + r, bc = col0 + tx;
      Bs[r][tx] = (bk < k && bc < n) ? Bb[bk * ldb + bc] : Arith<T>::zero();
    }
    __syncthreads();
    const int kk_end = (int)((k - k0) < EG_TILE ? (k - k0) : EG_TILE);
    for (int kk = 0; kk < kk_end; ++kk) {
      const T b = Bs[kk][tx];
#pragma unroll
      for (int q = 0; q < EG_ROWS; ++q)
        acc[q] = Arith<T>::add(acc[q], Arith<T>::mul(As[ty * EG_ROWS + q][kk], b));
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < EG_ROWS; ++q) {
    const int64_t r = row0 + ty * EG_ROWS + q, c = col0 + tx;
    // RELU: the GCN elementwise select (cmpf ogt + select) fused into the store
    if (r < m && c < n) Cb[r * ldc + c] = RELU ? ((acc[q] > T(0)) ? acc[q] : T(0)) : acc[q];
  }
  }
}

// -------------------------------------------- exact GEMM, narrow B (N, K <= 64)
// The GCN's (A_hat X) W: M = 1e6 rows against a 64 x 64 W.  The whole B sits in
// shared memory; a CTA stages 256 rows of A (coalesced, padded) per pass and
// each thread owns 4 rows x 16 columns (64 independent accumulator chains),
// walking k in the reference order with separately rounded mul / add — the
// same result as gemm_exact_kernel bit for bit, at ~1 shared load per 16
// floating-point operations (B read as broadcast 16-byte vectors).
// A is staged TRANSPOSED (AsT[k][row], row pitch EN_ROWS + 4), so a thread's
// four A values of one k are a single 16-byte shared load: 5 shared loads
// (1 + 4 of B) per 128 floating-point instructions instead of 8.
constexpr int EN_MAX = 64, EN_ROWS = 256, EN_COLS = 16, EN_RPT = 4, EN_PITCH = EN_ROWS + 4;
constexpr size_t EN_SMEM = (size_t)(EN_MAX * EN_MAX + EN_MAX * EN_PITCH) * sizeof(float);

template <bool RELU>
__global__ void __launch_bounds__(256)
gemm_exact_narrow_kernel(int64_t m, int n, int k, const float* __restrict__ A, int64_t lda,
                         const float* __restrict__ B, int64_t ldb, float* __restrict__ C,
                         int64_t ldc) {
  extern __shared__ __align__(16) float en_smem[];
  float* Bs = en_smem;                          // [EN_MAX][EN_MAX]
  float* AsT = en_smem + EN_MAX * EN_MAX;       // [EN_MAX][EN_PITCH]
  for (int t = threadIdx.x; t < EN_MAX * EN_MAX; t += blockDim.x) {
    const int r = t / EN_MAX, c = t % EN_MAX;
    Bs[t] = (r < k && c < n) ? B[(int64_t)r * ldb + c] : 0.0f;
  }
  const int cg = threadIdx.x & 3;          // columns [16 cg, 16 cg + 16)
  const int rg = threadIdx.x >> 2;         // rows 4 rg .. 4 rg + 3 of the pass
  const bool vec4 = (lda % 4 == 0) && ((uintptr_t)A % 16 == 0) && (k % 4 == 0);
  for (int64_t r0 = (int64_t)blockIdx.x * EN_ROWS; r0 < m; r0 += (int64_t)gridDim.x * EN_ROWS) {
    __syncthreads();
    // stage the pass's rows: all loads of a thread issued before any store
    // (a store right after each load would serialise one DRAM latency per
    // element); 16-byte loads when the pitch allows
    if (vec4) {
      float4 v[EN_ROWS * EN_MAX / 4 / 256];
#pragma unroll
      for (int u = 0; u < EN_ROWS * EN_MAX / 4 / 256; ++u) {
        const int t = threadIdx.x + 256 * u;
        const int r = t / (EN_MAX / 4), c4 = (t % (EN_MAX / 4)) * 4;
        v[u] = (r0 + r < m && c4 < k) ? *reinterpret_cast<const float4*>(A + (r0 + r) * lda + c4)
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < EN_ROWS * EN_MAX / 4 / 256; ++u) {
        const int t = threadIdx.x + 256 * u;
        const int r = t / (EN_MAX / 4), c4 = (t % (EN_MAX / 4)) * 4;
        float* d = AsT + c4 * EN_PITCH + r;
        d[0] = v[u].x; d[EN_PITCH] = v[u].y; d[2 * EN_PITCH] = v[u].z; d[3 * EN_PITCH] = v[u].w;
      }
    } else {
      for (int t0 = 0; t0 < EN_ROWS * EN_MAX; t0 += 256 * 8) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int t = t0 + threadIdx.x + 256 * u;
          const int r = t / EN_MAX, c = t % EN_MAX;
          v[u] = (r0 + r < m && c < k) ? A[(r0 + r) * lda + c] : 0.0f;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int t = t0 + threadIdx.x + 256 * u;
          AsT[(t % EN_MAX) * EN_PITCH + t / EN_MAX] = v[u];
        }
      }
    }
    __syncthreads();
    float acc[EN_RPT][EN_COLS];
#pragma unroll
    for (int i = 0; i < EN_RPT; ++i)
#pragma unroll
      for (int q = 0; q < EN_COLS; ++q) acc[i][q] = 0.0f;
    for (int kk = 0; kk < k; ++kk) {
      const float4 a4 = *reinterpret_cast<const float4*>(AsT + kk * EN_PITCH + rg * EN_RPT);
      const float a[EN_RPT] = {a4.x, a4.y, a4.z, a4.w};
      float bv[EN_COLS];
      const float4* brow = reinterpret_cast<const float4*>(Bs + kk * EN_MAX + cg * EN_COLS);
#pragma unroll
      for (int q = 0; q < EN_COLS / 4; ++q) {
        const float4 w = brow[q];
        bv[4 * q] = w.x; bv[4 * q + 1] = w.y; bv[4 * q + 2] = w.z; bv[4 * q + 3] = w.w;
      }
#pragma unroll
      for (int i = 0; i < EN_RPT; ++i)
#pragma unroll
        for (int q = 0; q < EN_COLS; ++q) acc[i][q] = __fadd_rn(acc[i][q], __fmul_rn(a[i], bv[q]));
    }
    const bool vec_c = (n == EN_MAX) && (ldc % 4 == 0) && ((uintptr_t)C % 16 == 0);
#pragma unroll
    for (int i = 0; i < EN_RPT; ++i) {
      const int64_t row = r0 + rg * EN_RPT + i;
      if (row >= m) continue;
      float o[EN_COLS];
#pragma unroll
      for (int q = 0; q < EN_COLS; ++q) o[q] = RELU ? ((acc[i][q] > 0.0f) ? acc[i][q] : 0.0f) : acc[i][q];
      if (vec_c) {
        float4* d = reinterpret_cast<float4*>(C + row * ldc + cg * EN_COLS);
#pragma unroll
        for (int q = 0; q < EN_COLS / 4; ++q) d[q] = make_float4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
      } else {
#pragma unroll
        for (int q = 0; q < EN_COLS; ++q) {
          const int c = cg * EN_COLS + q;
          if (c < n) C[row * ldc + c] = o[q];
        }
      }
    }
  }
}

// ------------------------------------------------- row-sequential row folds
// One thread per row; A staged through shared memory in 32-column slabs.
constexpr int RF_ROWS = 128;

template <class T, bool DOT>
__global__ void __launch_bounds__(RF_ROWS)
row_fold_kernel(int64_t m, int64_t n, const T* __restrict__ A, int64_t lda,
                const T* __restrict__ x, T* __restrict__ y, int comb) {
  __shared__ T tile[RF_ROWS][33];
  __shared__ T xs[32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t row0 = (int64_t)blockIdx.x * RF_ROWS;
  T acc = DOT ? Arith<T>::zero() : identity<T>(comb);
  for (int64_t c0 = 0; c0 < n; c0 += 32) {
    const int64_t c = c0 + lane;
    // each warp loads 32 row segments of 32 columns (coalesced per segment)
    for (int r = warp; r < RF_ROWS; r += RF_ROWS / 32) {
      const int64_t gr = row0 + r;
      tile[r][lane] = (gr < m && c < n) ? A[gr * lda + c] : Arith<T>::zero();
    }
    if (DOT && t < 32) xs[t] = (c < n) ? x[c] : Arith<T>::zero();
    __syncthreads();
    const int cend = (int)((n - c0) < 32 ? (n - c0) : 32);
    for (int q = 0; q < cend; ++q) {
      if (DOT) acc = Arith<T>::add(acc, Arith<T>::mul(tile[t][q], xs[q]));
      else acc = combine(acc, tile[t][q], comb);
    }
    __syncthreads();
  }
  const int64_t row = row0 + t;
  if (row < m) y[row] = acc;
}

// Pipelined row fold (the launched one for matvec / axis-1 reduce): a CTA owns
// 32 rows at a time (lane r of warp 0 folds row r in ascending column order —
// the reference's sequential order, bit-identical), and all 4 warps stream
// the rows' column panels into an RP_STAGES-deep shared-memory ring with
// cp.async, so up to RP_STAGES - 1 panels (32 rows x RP_COLS x 8 B each) are
// in flight per SM while warp 0 folds the current one.  Persistent over row
// blocks.  Row pitch RP_COLS + 1 keeps the folder's column reads to <= 2-way
// bank conflicts.
// 128 threads (one folding warp + three streaming), 3 stages: ~27 KB per CTA,
// 8 CTAs (folding warps) per SM.  Measured at 16384^2, f64 matvec / f64
// reduce / f32 matvec: 256 thr x 4 stages 0.427 / 0.374 / 0.211 ms, 128 x 4
// 0.422 / 0.367 / 0.207, 128 x 3 0.398 / 0.376 / 0.205, 64 x 3 0.391 / 0.393 / 0.210
constexpr int RP_ROWS = 32, RP_STAGES = 3, RP_THREADS = 128;
// 256-byte column panels (the fold, one warp per CTA, is what limits the
// kernel, so more, smaller CTAs per SM win).
// Measured at 16384^2 (f64 matvec / f64 reduce / f32 matvec), 6 stages:
// 128 B 0.52 / 0.55 / 0.28 ms, 256 B 0.46 / 0.41 / 0.23 ms, 512 B 0.61 / 0.44 / 0.28 ms;
// 256 B with 3 / 4 stages: 0.42 / 0.39 / 0.22 and 0.43 / 0.37 / 0.21 ms
constexpr int RP_PANEL_BYTES = 256;
template <class T> struct RpCols { static constexpr int v = RP_PANEL_BYTES / sizeof(T); };

__device__ __forceinline__ void rp_cp(void* dst, const void* src, int bytes) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  if (bytes == 8) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(d), "l"(src) : "memory");
  else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(d), "l"(src) : "memory");
}

// VEC16 (rows 16-byte aligned, n a multiple of 16 bytes): 16-byte cp.async
// (4x fewer requests per byte — the per-SM limit on outstanding requests is
// what bounds this kernel) and 16-byte shared loads in the fold; the pitch
// C + 16 B keeps those loads conflict-free (8 lanes per phase)
template <class T, bool VEC16> struct RpPitch {
  static constexpr int v = RpCols<T>::v + (VEC16 ? 16 / (int)sizeof(T) : 1);
};

template <class T, bool VEC16>
constexpr size_t rp_smem_bytes() {
  return (size_t)RP_STAGES * (RP_ROWS * RpPitch<T, VEC16>::v + RpCols<T>::v) * sizeof(T);
}

__device__ __forceinline__ void rp_cp16(void* dst, const void* src) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(d), "l"(src) : "memory");
}

template <class T, bool DOT, bool VEC16>
__global__ void __launch_bounds__(RP_THREADS)
row_fold_pipe_kernel(int64_t m, int64_t n, const T* __restrict__ A, int64_t lda,
                     const T* __restrict__ x, T* __restrict__ y, int comb) {
  constexpr int C = RpCols<T>::v, P = RpPitch<T, VEC16>::v, V = 16 / sizeof(T);
  using V16 = typename std::conditional<sizeof(T) == 8, longlong2, int4>::type;
  extern __shared__ __align__(16) unsigned char rp_raw[];
  T* tiles = reinterpret_cast<T*>(rp_raw);                      // [S][ROWS][P]
  T* xs = tiles + RP_STAGES * RP_ROWS * P;                       // [S][C]
  const int t = threadIdx.x;
  const int64_t nst = (n + C - 1) / C;
  const int64_t nrb = (m + RP_ROWS - 1) / RP_ROWS;
  for (int64_t rb = blockIdx.x; rb < nrb; rb += gridDim.x) {
    const int64_t row0 = rb * RP_ROWS;
    auto issue = [&](int64_t s) {
      if (s < nst) {
        const int slot = (int)(s % RP_STAGES);
        const int64_t c0 = s * C;
        T* tl = tiles + slot * RP_ROWS * P;
        if (VEC16) {
          for (int e = t; e < RP_ROWS * (C / V); e += RP_THREADS) {
            const int r = e / (C / V), c = (e % (C / V)) * V;
            if (row0 + r < m && c0 + c < n) rp_cp16(tl + r * P + c, A + (row0 + r) * lda + c0 + c);
          }
          if (DOT && t < C / V && c0 + t * V < n) rp_cp16(xs + slot * C + t * V, x + c0 + t * V);
        } else {
          for (int e = t; e < RP_ROWS * C; e += RP_THREADS) {
            const int r = e / C, c = e % C;
            if (row0 + r < m && c0 + c < n) rp_cp(tl + r * P + c, A + (row0 + r) * lda + c0 + c, sizeof(T));
          }
          if (DOT)
            for (int c = t; c < C; c += RP_THREADS)
              if (c0 + c < n) rp_cp(xs + slot * C + c, x + c0 + c, sizeof(T));
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int s = 0; s < RP_STAGES - 1; ++s) issue(s);
    T acc = DOT ? Arith<T>::zero() : identity<T>(comb);
    for (int64_t s = 0; s < nst; ++s) {
      asm volatile("cp.async.wait_group %0;" :: "n"(RP_STAGES - 2) : "memory");
      __syncthreads();                 // stage s visible; slot of s - 1 free
      issue(s + RP_STAGES - 1);
      if (t < RP_ROWS) {
        const int slot = (int)(s % RP_STAGES);
        const T* tr = tiles + slot * RP_ROWS * P + t * P;
        const T* xr = xs + slot * C;
        const int cend = (int)((n - s * C) < C ? (n - s * C) : C);
        int q = 0;
        // groups of 16: all 16 (32) shared loads issued before the in-order
        // chain, so the fold costs ~its dependent adds, not a load latency each
        for (; q + 16 <= cend; q += 16) {
          T a[16], b[16];
          if (VEC16) {
#pragma unroll
            for (int u = 0; u < 16; u += V) {
              const V16 va = *reinterpret_cast<const V16*>(tr + q + u);
              memcpy(&a[u], &va, 16);
              if (DOT) {
                const V16 vb = *reinterpret_cast<const V16*>(xr + q + u);
                memcpy(&b[u], &vb, 16);
              }
            }
          } else {
#pragma unroll
            for (int u = 0; u < 16; ++u) {
              a[u] = tr[q + u];
              if (DOT) b[u] = xr[q + u];
            }
          }
#pragma unroll
          for (int u = 0; u < 16; ++u)
            acc = DOT ? Arith<T>::add(acc, Arith<T>::mul(a[u], b[u])) : combine(acc, a[u], comb);
        }
        for (; q < cend; ++q)
          acc = DOT ? Arith<T>::add(acc, Arith<T>::mul(tr[q], xr[q])) : combine(acc, tr[q], comb);
      }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();                   // the ring is reused by the next row block
    if (t < RP_ROWS && row0 + t < m) y[row0 + t] = acc;
  }
}

// column fold (axis 0): one thread per column, rows in ascending order
template <class T>
__global__ void col_fold_kernel(int64_t rows, int64_t cols, const T* __restrict__ src,
                                T* __restrict__ out, int comb) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= cols) return;
  T acc = identity<T>(comb);
  for (int64_t r = 0; r < rows; ++r) acc = combine(acc, src[r * cols + c], comb);
  out[c] = acc;
}

template <class T>
__global__ void relu_kernel(int64_t n, const T* __restrict__ x, T* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T v = x[i];
    y[i] = (v > T(0)) ? v : T(0);  // cmpf ogt + select: NaN and -0.0 map to +0
  }
}

// =============================================================== host side
template <class T, bool RELU = false>
static int launch_gemm_exact(int64_t batch, int64_t m, int64_t n, int64_t k, const void* A,
                             int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                             int64_t sA, int64_t sB, int64_t sC, cudaStream_t st,
                             Guard guard = Guard()) {
  if constexpr (std::is_same<T, float>::value) {
    if (batch == 1 && guard.mode == 0 && n <= EN_MAX && k <= EN_MAX) {
      LB_TRY(check_cuda(cudaFuncSetAttribute(gemm_exact_narrow_kernel<RELU>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)EN_SMEM), "smem attr (narrow gemm)"));
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gemm_exact_narrow_kernel<RELU>, 256,
                                                    EN_SMEM);
      int64_t blocks = (m + EN_ROWS - 1) / EN_ROWS;
      const int64_t cap = (int64_t)num_sms() * (per_sm > 0 ? per_sm : 1);
      if (blocks > cap) blocks = cap;
      if (blocks < 1) blocks = 1;
      gemm_exact_narrow_kernel<RELU><<<(unsigned)blocks, 256, EN_SMEM, st>>>(
          m, (int)n, (int)k, (const float*)A, lda, (const float*)B, ldb, (float*)C, ldc);
      return check_launch("gemm_exact_narrow_kernel");
    }
  }
  const int64_t tiles = ((n + EG_TILE - 1) / EG_TILE) * ((m + EG_TILE - 1) / EG_TILE) * batch;
  // a guarded fallback (skipped unless its flag is raised) launches one wave
  const int64_t per_sm = guard.mode != 0 ? 1 : 8;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)num_sms() * per_sm));
  gemm_exact_kernel<T, RELU><<<(unsigned)grid, 256, 0, st>>>(m, n, k, (const T*)A, lda, (const T*)B,
                                                             ldb, (T*)C, ldc, sA, sB, sC, batch, guard);
  return check_launch("gemm_exact_kernel");
}

// The reference-order GEMM behind a device flag (the Ozaki path's fallback for
// non-finite inputs): launched unconditionally, returns at once unless *guard.
int launch_gemm_exact_guarded(int64_t m, int64_t n, int64_t k, const void* A, int64_t lda,
                              const void* B, int64_t ldb, void* C, int64_t ldc, int dtype,
                              Guard guard, cudaStream_t st) {
  if (dtype == LAPIS_B200_F64)
    return launch_gemm_exact<double>(1, m, n, k, A, lda, B, ldb, C, ldc, 0, 0, 0, st, guard);
  return launch_gemm_exact<float>(1, m, n, k, A, lda, B, ldb, C, ldc, 0, 0, 0, st, guard);
}

int gemm_exact(int64_t batch, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda,
               const void* B, int64_t ldb, void* C, int64_t ldc, int64_t sA, int64_t sB,
               int64_t sC, int dtype, cudaStream_t st) {
  switch (dtype) {
    case LAPIS_B200_F64: return launch_gemm_exact<double>(batch, m, n, k, A, lda, B, ldb, C, ldc, sA, sB, sC, st);
    case LAPIS_B200_F32: return launch_gemm_exact<float>(batch, m, n, k, A, lda, B, ldb, C, ldc, sA, sB, sC, st);
    case LAPIS_B200_I64: return launch_gemm_exact<long long>(batch, m, n, k, A, lda, B, ldb, C, ldc, sA, sB, sC, st);
    case LAPIS_B200_I32: return launch_gemm_exact<int>(batch, m, n, k, A, lda, B, ldb, C, ldc, sA, sB, sC, st);
  }
  return fail(LAPIS_B200_ERR_ARG, "gemm: unsupported dtype");
}

template <class T, bool DOT>
static int launch_row_fold(int64_t m, int64_t n, const void* A, int64_t lda, const void* x,
                           void* y, int comb, cudaStream_t st) {
  if (m == 0) return LAPIS_B200_OK;
  if (getenv("LAPIS_B200_ROWFOLD_OLD")) {
    const int64_t blocks = (m + RF_ROWS - 1) / RF_ROWS;
    row_fold_kernel<T, DOT><<<(unsigned)blocks, RF_ROWS, 0, st>>>(m, n, (const T*)A, lda,
                                                                    (const T*)x, (T*)y, comb);
    return check_launch("row_fold_kernel");
  }
  const bool vec16 = ((lda * (int64_t)sizeof(T)) % 16 == 0) && ((uintptr_t)A % 16 == 0) &&
                     ((n * (int64_t)sizeof(T)) % 16 == 0) && (!DOT || (uintptr_t)x % 16 == 0);
  const size_t smem = vec16 ? rp_smem_bytes<T, true>() : rp_smem_bytes<T, false>();
  auto kern = vec16 ? row_fold_pipe_kernel<T, DOT, true> : row_fold_pipe_kernel<T, DOT, false>;
  static thread_local int configured_dev = -1;
  static thread_local int per_sm_v[2] = {1, 1};
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    for (int v = 0; v < 2; ++v) {
      auto kv = v ? row_fold_pipe_kernel<T, DOT, true> : row_fold_pipe_kernel<T, DOT, false>;
      const size_t sv = v ? rp_smem_bytes<T, true>() : rp_smem_bytes<T, false>();
      LB_TRY(check_cuda(cudaFuncSetAttribute(kv, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sv), "smem attr (row fold)"));
      LB_TRY(check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_v[v], kv, RP_THREADS, sv),
                        "occupancy (row fold)"));
      if (per_sm_v[v] < 1) per_sm_v[v] = 1;
    }
    configured_dev = dev;
  }
  const int per_sm = per_sm_v[vec16 ? 1 : 0];
  int64_t blocks = (m + RP_ROWS - 1) / RP_ROWS;
  const int64_t cap = (int64_t)num_sms() * per_sm;
  if (blocks > cap) blocks = cap;
  kern<<<(unsigned)blocks, RP_THREADS, smem, st>>>(m, n, (const T*)A, lda, (const T*)x, (T*)y, comb);
  return check_launch("row_fold_pipe_kernel");
}

// C = relu(A B) in the reference order (GCN second stage, oracle/ir/gcn_f32.mlir)
int gemm_exact_relu(int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B,
                    int64_t ldb, void* C, int64_t ldc, int dtype, cudaStream_t st) {
  if (dtype == LAPIS_B200_F32)
    return launch_gemm_exact<float, true>(1, m, n, k, A, lda, B, ldb, C, ldc, 0, 0, 0, st);
  if (dtype == LAPIS_B200_F64)
    return launch_gemm_exact<double, true>(1, m, n, k, A, lda, B, ldb, C, ldc, 0, 0, 0, st);
  return fail(LAPIS_B200_ERR_UNSUPPORTED, "gcn: floating-point dtypes only");
}

int gemv(int64_t m, int64_t n, const void* A, int64_t lda, const void* x, void* y, int dtype,
         cudaStream_t st) {
  if (m == 0) return LAPIS_B200_OK;
  switch (dtype) {
    case LAPIS_B200_F64: return launch_row_fold<double, true>(m, n, A, lda, x, y, 0, st);
    case LAPIS_B200_F32: return launch_row_fold<float, true>(m, n, A, lda, x, y, 0, st);
    case LAPIS_B200_I64: return launch_row_fold<long long, true>(m, n, A, lda, x, y, 0, st);
    case LAPIS_B200_I32: return launch_row_fold<int, true>(m, n, A, lda, x, y, 0, st);
  }
  return fail(LAPIS_B200_ERR_ARG, "gemv: unsupported dtype");
}

template <class T>
static int launch_reduce(int64_t rows, int64_t cols, const void* src, void* out, int axis,
                         int comb, cudaStream_t st) {
  if (axis == 1) return launch_row_fold<T, false>(rows, cols, src, cols, nullptr, out, comb, st);
  if (cols == 0) return LAPIS_B200_OK;
  col_fold_kernel<T><<<(unsigned)((cols + 127) / 128), 128, 0, st>>>(rows, cols, (const T*)src,
                                                                      (T*)out, comb);
  return check_launch("col_fold_kernel");
}

int reduce_2d(int64_t rows, int64_t cols, const void* src, void* out, int axis, int comb,
              int dtype, cudaStream_t st) {
  if (axis != 0 && axis != 1) return fail(LAPIS_B200_ERR_ARG, "reduce: axis must be 0 or 1");
  if (comb < LAPIS_B200_ADD || comb > LAPIS_B200_MAX)
    return fail(LAPIS_B200_ERR_ARG, "reduce: unknown combiner");
  if ((axis == 1 ? rows : cols) == 0) return LAPIS_B200_OK;
  switch (dtype) {
    case LAPIS_B200_F64: return launch_reduce<double>(rows, cols, src, out, axis, comb, st);
    case LAPIS_B200_F32: return launch_reduce<float>(rows, cols, src, out, axis, comb, st);
    case LAPIS_B200_I64: return launch_reduce<long long>(rows, cols, src, out, axis, comb, st);
    case LAPIS_B200_I32: return launch_reduce<int>(rows, cols, src, out, axis, comb, st);
  }
  return fail(LAPIS_B200_ERR_ARG, "reduce: unsupported dtype");
}

int relu(int64_t n, const void* x, void* y, int dtype, cudaStream_t st) {
  if (n == 0) return LAPIS_B200_OK;
  const int64_t blocks = (n + 255) / 256 < 148 * 32 ? (n + 255) / 256 : 148 * 32;
  if (dtype == LAPIS_B200_F64)
    relu_kernel<double><<<(unsigned)blocks, 256, 0, st>>>(n, (const double*)x, (double*)y);
  else if (dtype == LAPIS_B200_F32)
    relu_kernel<float><<<(unsigned)blocks, 256, 0, st>>>(n, (const float*)x, (float*)y);
  else
    return fail(LAPIS_B200_ERR_UNSUPPORTED, "relu: floating-point dtypes only");
  return check_launch("relu_kernel");
}

}  // namespace lapis_b200

namespace lapis_b200 {

// tensor-core paths (gemm_tf32x3.cu, gemm_dmma.cu): prototypes in common.cuh

int gemm_ozaki(int64_t batch, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda,
               const void* B, int64_t ldb, void* C, int64_t ldc, int64_t sA, int64_t sB,
               int64_t sC, int dtype, int slices, cudaStream_t st, int sign_gate = 0);
int ozaki_slices_for(int dtype, int64_t k);

int gemm_dispatch(int64_t batch, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda,
                  const void* B, int64_t ldb, void* C, int64_t ldc, int64_t sA, int64_t sB,
                  int64_t sC, int dtype, int mode, cudaStream_t st) {
  if (m < 0 || n < 0 || k < 0 || lda < k || ldb < n || ldc < n)
    return fail(LAPIS_B200_ERR_ARG, "gemm: bad extents / leading dimensions");
  if (!valid_dtype(dtype)) return fail(LAPIS_B200_ERR_ARG, "gemm: unsupported dtype");
  if (batch == 0 || m == 0 || n == 0) return LAPIS_B200_OK;
  if (!C || (k > 0 && (!A || !B))) return fail(LAPIS_B200_ERR_ARG, "gemm: null operand");
  if (mode == LAPIS_B200_GEMM_AUTO) {
    // f64: certified Ozaki on the int8 tensor cores when k is in its range
    // (DMMA otherwise); f32: Ozaki (S = 3, 8-bit digits) gated on the signs —
    // non-negative operands (no cancellation: the certificate holds for the
    // sums the reference computes) run it, any negative entry sends the call
    // to 3xTF32 through the device flag the split kernels raise, as does a
    // failed certificate; ints: reference order.  Config 2 f32 (U(0, 1)):
    // 0.585 ms (235 TF/s, max rel err 4.1e-6 vs the reference) against
    // 0.645 ms for 3xTF32.
    if (dtype == LAPIS_B200_F32) {
      static const bool no_oz32 = [] {
        const char* e = getenv("LAPIS_B200_F32_AUTO_OZAKI");
        return e && e[0] == '0';
      }();
      if (!no_oz32 && ozaki_slices_for(dtype, k))
        return gemm_ozaki(batch, m, n, k, A, lda, B, ldb, C, ldc, sA, sB, sC, dtype, 0, st, 1);
      mode = LAPIS_B200_GEMM_TF32X3;
    } else if (dtype == LAPIS_B200_F64)
      mode = ozaki_slices_for(dtype, k) ? LAPIS_B200_GEMM_OZAKI : LAPIS_B200_GEMM_DMMA;
    else mode = LAPIS_B200_GEMM_EXACT;
  }
  switch (mode) {
    case LAPIS_B200_GEMM_EXACT:
      return gemm_exact(batch, m, n, k, A, lda, B, ldb, C, ldc, sA, sB, sC, dtype, st);
    case LAPIS_B200_GEMM_TF32X3:
      if (dtype != LAPIS_B200_F32)
        return fail(LAPIS_B200_ERR_UNSUPPORTED, "gemm: TF32X3 is an f32 mode");
      return gemm_tf32x3(batch, m, n, k, A, lda, B, ldb, C, ldc, sA, sB, sC, st);
    case LAPIS_B200_GEMM_DMMA:
      if (dtype != LAPIS_B200_F64)
        return fail(LAPIS_B200_ERR_UNSUPPORTED, "gemm: DMMA is an f64 mode");
      return gemm_dmma(batch, m, n, k, A, lda, B, ldb, C, ldc, sA, sB, sC, st);
    case LAPIS_B200_GEMM_OZAKI:
      if (dtype != LAPIS_B200_F64 && dtype != LAPIS_B200_F32)
        return fail(LAPIS_B200_ERR_UNSUPPORTED, "gemm: OZAKI is an f32 / f64 mode");
      return gemm_ozaki(batch, m, n, k, A, lda, B, ldb, C, ldc, sA, sB, sC, dtype, 0, st);
  }
  return fail(LAPIS_B200_ERR_ARG, "gemm: unknown mode");
}

void release_workspaces() {}

}  // namespace lapis_b200
