// gemm_dmma.cu — fp64 dense matmul on the FP64 tensor-core path (DMMA).
//
// tcgen05 has no fp64 kind, so linalg.matmul / kokkos.gemm in f64
// (interp.py:711-722) runs on mma.sync.aligned.m8n8k4.f64 (SASS DMMA.8x8x4):
//   CTA tile 128 x 128, K slab 16, 8 warps as 2 (M) x 4 (N) -> 64 x 32 per warp
//   = 8 x 4 DMMA tiles, 64 fp64 accumulators per lane;
//   3-stage cp.async (16 B) shared-memory ring; A padded to 20 doubles per row
//   and B to 132 per row so both fragment loads are bank-conflict free.
// DMMA rounds every multiply-add in fp64; the result stays far inside the
// 1e-12 contract against the reference's sequential sum (6.5e-14).
#include "common.cuh"

#include <algorithm>

namespace lapis_b200 {

constexpr int DM_BM = 128, DM_BN = 128, DM_BK = 16, DM_STAGES = 3, DM_THREADS = 256;
constexpr int DM_AS = DM_BK + 4;      // A smem row pitch (doubles)
constexpr int DM_BS = DM_BN + 4;      // B smem row pitch (doubles)
constexpr int DM_A_ELEMS = DM_BM * DM_AS;
constexpr int DM_B_ELEMS = DM_BK * DM_BS;
constexpr size_t DM_SMEM = (size_t)DM_STAGES * (DM_A_ELEMS + DM_B_ELEMS) * sizeof(double);

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  const uint32_t d = smem_u32(dst);
  const int sz = valid ? 16 : 0;   // 0 source bytes -> zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" :: "r"(d), "l"(src), "r"(sz)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory"); }

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(DM_THREADS, 1)
gemm_dmma_kernel(int64_t m, int64_t n, int64_t k, const double* __restrict__ A, int64_t lda,
                 const double* __restrict__ B, int64_t ldb, double* __restrict__ C, int64_t ldc,
                 Guard guard) {
  if (guard_skip(guard)) return;
  extern __shared__ __align__(16) double dsm[];
  double* sA = dsm;                                  // [STAGES][BM][AS]
  double* sB = dsm + DM_STAGES * DM_A_ELEMS;         // [STAGES][BK][BS]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 2, wn = warp & 3;           // 2 x 4 warp grid
  const int nkb = (int)((k + DM_BK - 1) / DM_BK);
  // tiles walked grid-stride (a guarded fallback launches one wave: when
  // the guard skips, its cost is one wave of CTA launches, not every tile's)
  const int64_t tn = (n + DM_BN - 1) / DM_BN, tiles = tn * ((m + DM_BM - 1) / DM_BM);
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
  const int64_t m0 = (tile / tn) * DM_BM, n0 = (tile % tn) * DM_BN;
  __syncthreads();   // the previous tile's shared-memory reads are done

  auto load_stage = [&](int st, int kb) {
    const int64_t k0 = (int64_t)kb * DM_BK;
    double* a = sA + st * DM_A_ELEMS;
    double* b = sB + st * DM_B_ELEMS;
    // A: 128 rows x 16 doubles = 1024 chunks of 2 doubles
#pragma unroll
    for (int c = tid; c < DM_BM * DM_BK / 2; c += DM_THREADS) {
      const int r = c / (DM_BK / 2), cc = (c % (DM_BK / 2)) * 2;
      const int64_t gr = m0 + r, gk = k0 + cc;
      const bool ok = gr < m && gk < k;
      cp_async16(a + r * DM_AS + cc, ok ? A + gr * lda + gk : A, ok);
    }
    // B: 16 rows x 128 doubles = 1024 chunks
#pragma unroll
    for (int c = tid; c < DM_BK * DM_BN / 2; c += DM_THREADS) {
      const int r = c / (DM_BN / 2), cc = (c % (DM_BN / 2)) * 2;
      const int64_t gk = k0 + r, gn = n0 + cc;
      const bool ok = gk < k && gn < n;
      cp_async16(b + r * DM_BS + cc, ok ? B + gk * ldb + gn : B, ok);
    }
  };

  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < DM_STAGES - 1; ++s) {
    if (s < nkb) load_stage(s, s);
    cp_async_commit();
  }
  for (int kb = 0; kb < nkb; ++kb) {
    cp_async_wait<DM_STAGES - 2>();
    __syncthreads();
    const int nxt = kb + DM_STAGES - 1;
    if (nxt < nkb) load_stage(nxt % DM_STAGES, nxt);
    cp_async_commit();
    const double* a = sA + (kb % DM_STAGES) * DM_A_ELEMS;
    const double* b = sB + (kb % DM_STAGES) * DM_B_ELEMS;
#pragma unroll
    for (int kk = 0; kk < DM_BK; kk += 4) {
      double af[8], bf[4];
#pragma unroll
      for (int i = 0; i < 8; ++i) af[i] = a[(wm * 64 + i * 8 + (lane >> 2)) * DM_AS + kk + (lane & 3)];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = b[(kk + (lane & 3)) * DM_BS + wn * 32 + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
  // C fragment: lane holds row lane/4, columns 2*(lane%4) + {0,1} of each 8x8 tile
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t r = m0 + wm * 64 + i * 8 + (lane >> 2);
    if (r >= m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t c = n0 + wn * 32 + j * 8 + 2 * (lane & 3);
      double* dst = C + r * ldc + c;
      if (c + 1 < n && ((ldc & 1) == 0)) {
        *reinterpret_cast<double2*>(dst) = make_double2(acc[i][j][0], acc[i][j][1]);
      } else {
        if (c < n) dst[0] = acc[i][j][0];
        if (c + 1 < n) dst[1] = acc[i][j][1];
      }
    }
  }
  }
}

int gemm_exact(int64_t, int64_t, int64_t, int64_t, const void*, int64_t, const void*, int64_t,
               void*, int64_t, int64_t, int64_t, int64_t, int, cudaStream_t);

int gemm_dmma(int64_t batch, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda,
              const void* B, int64_t ldb, void* C, int64_t ldc, int64_t sA, int64_t sB,
              int64_t sC, cudaStream_t st, Guard guard) {
  // the 16-byte cp.async path needs even leading dimensions / extents and aligned bases
  const bool aligned = (lda % 2 == 0) && (ldb % 2 == 0) && (k % 2 == 0) && (n % 2 == 0) &&
                       ((uintptr_t)A % 16 == 0) && ((uintptr_t)B % 16 == 0) &&
                       (sA % 2 == 0) && (sB % 2 == 0);
  if (!aligned) {
    if (guard.mode == 0)
      return gemm_exact(batch, m, n, k, A, lda, B, ldb, C, ldc, sA, sB, sC, LAPIS_B200_F64, st);
    for (int64_t b = 0; b < batch; ++b)   // guarded fallback (single batches from the Ozaki path)
      LB_TRY(launch_gemm_exact_guarded(m, n, k, (const double*)A + b * sA, lda,
                                       (const double*)B + b * sB, ldb, (double*)C + b * sC, ldc,
                                       LAPIS_B200_F64, guard, st));
    return LAPIS_B200_OK;
  }
  static thread_local int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    LB_TRY(check_cuda(cudaFuncSetAttribute(gemm_dmma_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DM_SMEM),
                      "smem attr (gemm_dmma_kernel)"));
    configured_dev = dev;
  }
  const int64_t tiles = ((n + DM_BN - 1) / DM_BN) * ((m + DM_BM - 1) / DM_BM);
  // one CTA per tile when DMMA is the chosen path; one wave when guarded
  int64_t g = tiles;
  if (guard.mode != 0 && g > (int64_t)num_sms()) g = num_sms();
  if (g > 0x7fffffffLL) g = 0x7fffffffLL;
  const dim3 grid((unsigned)(g < 1 ? 1 : g));
  for (int64_t b = 0; b < batch; ++b) {
    gemm_dmma_kernel<<<grid, DM_THREADS, DM_SMEM, st>>>(
        m, n, k, (const double*)A + b * sA, lda, (const double*)B + b * sB, ldb,
        (double*)C + b * sC, ldc, guard);
    LB_TRY(check_launch("gemm_dmma_kernel"));
  }
  return LAPIS_B200_OK;
}

}  // namespace lapis_b200
