// gemm_tf32x3.cu — fp32 dense matmul on the 5th-generation tensor cores.
//
// C = A * B (row-major, LayoutRight) for linalg.matmul / kokkos.gemm
// (interp.py:711-722, runtime_header.py:249-266) at fp32 accuracy with TF32
// tensor-core math ("3xTF32"): every operand is split into a TF32 head and a
// TF32 tail, a = a_hi + a_lo with a_hi = rna_tf32(a), a_lo = rna_tf32(a - a_hi),
// and C = A_lo*B_hi + A_hi*B_lo + A_hi*B_hi accumulated in fp32 (the dropped
// A_lo*B_lo term is ~2^-22 relative).  Plain 1xTF32 misses the 1e-5 contract
// (SURVEY A.7); 3xTF32 matches fp32 SIMT accuracy.
//
// Kernel shape (sm_100a, one CTA per SM, persistent over 128x256 output tiles):
//   warp 0      TMA producer: cp.async.bulk.tensor 2-D loads of 128x32 A and
//               256x32 B^T fp32 boxes (SWIZZLE_128B) into a 4-stage ring,
//               completion on full[stage] (expect_tx)
//   warp 1      TMEM allocator + MMA issuer: one elected thread issues
//               tcgen05.mma.cta_group::1.kind::tf32 (M=128, N=256, K=8) from
//               shared-memory descriptors into a double-buffered TMEM
//               accumulator (2 x 256 columns); tcgen05.commit frees each stage
//               (empty[stage]) and publishes a finished tile (tmem_full[acc])
//   warps 2..5  epilogue: tcgen05.ld 32x32b.x16 (warp w reads TMEM lanes
//               32*(w%4)...), fp32 stores to C, then release the accumulator
//               (tmem_empty[acc]) so the MMA of the next tile overlaps.
// The k loop runs 3 phases per tile (lo*hi, hi*lo, hi*hi) over the split
// operands, i.e. a TF32 GEMM with K' = 3K.  The split (and the transpose that
// makes B K-major) is a bandwidth-bound prepass.
#include "common.cuh"
#include "tcgen05.cuh"

#include <algorithm>

namespace lapis_b200 {

constexpr int TG_BM = 128, TG_BN = 256, TG_BK = 32, TG_STAGES = 4, TG_UMMA_K = 8;
constexpr uint32_t TG_A_BYTES = TG_BM * TG_BK * 4;  // 16 KB
constexpr uint32_t TG_B_BYTES = TG_BN * TG_BK * 4;  // 32 KB
constexpr uint32_t TG_STAGE_BYTES = TG_A_BYTES + TG_B_BYTES;
constexpr uint32_t TG_TMEM_COLS = 512;
constexpr size_t TG_SMEM = (size_t)TG_STAGES * TG_STAGE_BYTES + 1024;

struct Tf32Params {
  int m, n, nk;       // nk = k blocks of TG_BK
  int num_m, num_n;   // tile grid
  float* C;
  int64_t ldc;
};

// instruction descriptor: D f32, A/B tf32, both K-major, N>>3, M>>4
__host__ __device__ constexpr uint32_t tf32_idesc(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

// ----------------------------------------------------------------------- kernel
// Accuracy note: the tensor core adds each MMA into the fp32 accumulator with
// truncation, so a single accumulator over K' = 3K terms drifts ~#MMA * 2^-25
// (3e-5 at 4096^3, outside the 1e-5 contract).  The k range is therefore cut
// into chunks of TG_KC k-blocks; each chunk is accumulated in TMEM (tail
// phases first, head*head last) and drained by the epilogue into round-to-
// nearest fp32 register sums, which bounds the drift to ~1e-6.
constexpr int TG_KC = 8;                 // k-blocks per chunk (256 of K)
constexpr int TG_EPI_WARPS = 8;          // two per TMEM lane group, 128 columns each
constexpr int TG_THREADS_V2 = 64 + TG_EPI_WARPS * 32;

__global__ void __launch_bounds__(TG_THREADS_V2, 1)
gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap tA_hi, const __grid_constant__ CUtensorMap tA_lo,
                   const __grid_constant__ CUtensorMap tB_hi, const __grid_constant__ CUtensorMap tB_lo,
                   Tf32Params p, Guard guard) {
  if (guard_skip(guard)) return;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[TG_STAGES], empty[TG_STAGES], tmem_full[2], tmem_empty[2];
  __shared__ uint32_t tmem_base_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int total = p.num_m * p.num_n;
  const int nchunks = (p.nk + TG_KC - 1) / TG_KC;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tA_hi); prefetch_tmap(&tA_lo); prefetch_tmap(&tB_hi); prefetch_tmap(&tB_lo);
    for (int s = 0; s < TG_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], TG_EPI_WARPS * 32);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(&tmem_base_slot)), "r"(TG_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
        const int mb = tile % p.num_m, nb = tile / p.num_m;
        for (int ch = 0; ch < nchunks; ++ch) {
          const int kb0 = ch * TG_KC, kb1 = min(kb0 + TG_KC, p.nk);
          for (int ph = 0; ph < 3; ++ph) {
            for (int kb = kb0; kb < kb1; ++kb) {
              mbar_wait(&empty[stage], phase ^ 1);
              uint8_t* sa = smem + stage * TG_STAGE_BYTES;
              uint8_t* sb = sa + TG_A_BYTES;
              mbar_arrive_expect_tx(&full[stage], TG_STAGE_BYTES);
              tma_load_2d(sa, ph == 0 ? &tA_lo : &tA_hi, kb * TG_BK, mb * TG_BM, &full[stage]);
              tma_load_2d(sb, ph == 1 ? &tB_lo : &tB_hi, kb * TG_BK, nb * TG_BN, &full[stage]);
              if (++stage == TG_STAGES) { stage = 0; phase ^= 1; }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------------------------------------------------- MMA issuer
      constexpr uint32_t idesc = tf32_idesc(TG_BM, TG_BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
        for (int ch = 0; ch < nchunks; ++ch) {
          const int kb0 = ch * TG_KC, kb1 = min(kb0 + TG_KC, p.nk);
          mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + (uint32_t)(acc * TG_BN);
          bool first = true;
          for (int ph = 0; ph < 3; ++ph) {
            for (int kb = kb0; kb < kb1; ++kb) {
              mbar_wait(&full[stage], phase);
              tc_fence_after();
              const uint8_t* sa = smem + stage * TG_STAGE_BYTES;
              const uint64_t adesc = smem_desc_sw128(sa);
              const uint64_t bdesc = smem_desc_sw128(sa + TG_A_BYTES);
#pragma unroll
              for (int kk = 0; kk < TG_BK / TG_UMMA_K; ++kk) {
                // advance the start address by kk * 32 bytes inside the 128-B swizzle atom
                tc_mma_tf32(d_tmem, adesc + (uint64_t)(kk * 2), bdesc + (uint64_t)(kk * 2),
                            idesc, first ? 0u : 1u);
                first = false;
              }
              tc_commit(&empty[stage]);
              if (++stage == TG_STAGES) { stage = 0; phase ^= 1; }
            }
          }
          tc_commit(&tmem_full[acc]);
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 2;                 // 0..7
    const int lg = warp & 3;                 // TMEM lane group this warp may access
    const int half = ew >> 2;                // columns [128*half, 128*half + 128)
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
      const int mb = tile % p.num_m, nb = tile / p.num_m;
      float sum[128];
#pragma unroll
      for (int q = 0; q < 128; ++q) sum[q] = 0.0f;
      for (int ch = 0; ch < nchunks; ++ch) {
        mbar_wait(&tmem_full[acc], acc_phase);
        tc_fence_after();
        const uint32_t tbase = tmem_base + ((uint32_t)(lg * 32) << 16) +
                               (uint32_t)(acc * TG_BN + half * 128);
#pragma unroll
        for (int c0 = 0; c0 < 128; c0 += 16) {
          uint32_t v[16];
          tmem_ld_x16(tbase + (uint32_t)c0, v);
#pragma unroll
          for (int q = 0; q < 16; ++q) sum[c0 + q] = __fadd_rn(sum[c0 + q], __uint_as_float(v[q]));
        }
        tc_fence_before();
        mbar_arrive(&tmem_empty[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
      const int row = mb * TG_BM + lg * 32 + lane;
      const int col0 = nb * TG_BN + half * 128;
      if (row < p.m) {
        float* crow = p.C + (int64_t)row * p.ldc;
        if (col0 + 128 <= p.n && (p.ldc % 4 == 0)) {
          float4* dst = reinterpret_cast<float4*>(crow + col0);
#pragma unroll
          for (int q = 0; q < 32; ++q)
            dst[q] = make_float4(sum[4 * q], sum[4 * q + 1], sum[4 * q + 2], sum[4 * q + 3]);
        } else {
#pragma unroll
          for (int q = 0; q < 128; ++q)
            if (col0 + q < p.n) crow[col0 + q] = sum[q];
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;"
                 :: "r"(tmem_base), "r"(TG_TMEM_COLS));
  }
}

// --------------------------------------------------------------- split prepass
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ float tf32_trunc(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xffffe000u);
}
// head / tail of the split: rawhi = 1 keeps the fp32 value as the head (the
// tensor core reads only its TF32 bits) and the tail is a - trunc(a)
__device__ __forceinline__ void tf32_split(float a, int rawhi, float& h, float& l) {
  if (rawhi) {
    h = a;
    l = tf32_rna(a - tf32_trunc(a));
  } else {
    h = tf32_rna(a);
    l = tf32_rna(a - h);
  }
}

// A [m, k] (lda) -> hi, lo [m, kp], zero padded for k <= j < kp
__global__ void split_rows_kernel(int64_t m, int64_t k, int64_t kp, const float* __restrict__ A,
                                  int64_t lda, float* __restrict__ hi, float* __restrict__ lo,
                                  Guard guard, int rawhi) {
  if (guard_skip(guard)) return;
  // a CTA per row (grid-stride), 4 consecutive elements per thread: 16-byte
  // loads when the row pitch allows, 16-byte stores (kp % 4 == 0), no
  // per-element 64-bit division
  const bool vec = (lda % 4 == 0) && ((uintptr_t)A % 16 == 0);
  for (int64_t i = blockIdx.x; i < m; i += gridDim.x) {
    const float* ar = A + i * lda;
    float4* hr = reinterpret_cast<float4*>(hi + i * kp);
    float4* lr = reinterpret_cast<float4*>(lo + i * kp);
    for (int64_t j4 = threadIdx.x; j4 < kp / 4; j4 += blockDim.x) {
      const int64_t j = 4 * j4;
      float4 a;
      if (vec && j + 3 < k) {
        a = *reinterpret_cast<const float4*>(ar + j);
      } else {
        a.x = j < k ? ar[j] : 0.0f;
        a.y = j + 1 < k ? ar[j + 1] : 0.0f;
        a.z = j + 2 < k ? ar[j + 2] : 0.0f;
        a.w = j + 3 < k ? ar[j + 3] : 0.0f;
      }
      float4 h, l;
      tf32_split(a.x, rawhi, h.x, l.x);
      tf32_split(a.y, rawhi, h.y, l.y);
      tf32_split(a.z, rawhi, h.z, l.z);
      tf32_split(a.w, rawhi, h.w, l.w);
      hr[j4] = h;
      lr[j4] = l;
    }
  }
}

// B [k, n] (ldb) -> hi, lo [n, kp] (transposed: K-major), zero padded
__global__ void split_transpose_kernel(int64_t k, int64_t n, int64_t kp, const float* __restrict__ B,
                                       int64_t ldb, float* __restrict__ hi, float* __restrict__ lo,
                                       Guard guard, int rawhi) {
  if (guard_skip(guard)) return;
  // 64 (k) x 64 (n) tile, 256 threads: coalesced 128-byte row loads, 8-byte
  // stores of consecutive k pairs (kp is a multiple of 4)
  __shared__ float tile[64][65];
  const int64_t k0 = (int64_t)blockIdx.y * 64, n0 = (int64_t)blockIdx.x * 64;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
  for (int r = ty; r < 64; r += 8) {
    const int64_t kk = k0 + r;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t nn = n0 + tx + 32 * h;
      tile[r][tx + 32 * h] = (kk < k && nn < n) ? B[kk * ldb + nn] : 0.0f;
    }
  }
  __syncthreads();
  const int64_t kk = k0 + 2 * tx;
  for (int r = ty; r < 64; r += 8) {
    const int64_t nn = n0 + r;
    if (nn < n && kk < kp) {
      const float a0 = tile[2 * tx][r], a1 = tile[2 * tx + 1][r];
      float h0, h1, l0, l1;
      tf32_split(a0, rawhi, h0, l0);
      tf32_split(a1, rawhi, h1, l1);
      *reinterpret_cast<float2*>(hi + nn * kp + kk) = make_float2(h0, h1);
      *reinterpret_cast<float2*>(lo + nn * kp + kk) = make_float2(l0, l1);
    }
  }
}

// tails only (RAW kernel): lo[i, j] = rna_tf32(a - trunc_tf32(a)) for
// j < cols, 0 for cols <= j < ldo; rows x cols with pitch lda -> pitch ldo
__global__ void tf32_tail_kernel(int64_t rows, int64_t cols, int64_t ldo, const float* __restrict__ A,
                                 int64_t lda, float* __restrict__ lo, Guard guard) {
  if (guard_skip(guard)) return;
  const bool vec = (lda % 4 == 0) && ((uintptr_t)A % 16 == 0);
  for (int64_t i = blockIdx.x; i < rows; i += gridDim.x) {
    const float* ar = A + i * lda;
    float4* lr = reinterpret_cast<float4*>(lo + i * ldo);
    for (int64_t j4 = threadIdx.x; j4 < ldo / 4; j4 += blockDim.x) {
      const int64_t j = 4 * j4;
      float4 a;
      if (vec && j + 3 < cols) {
        a = *reinterpret_cast<const float4*>(ar + j);
      } else {
        a.x = j < cols ? ar[j] : 0.0f;
        a.y = j + 1 < cols ? ar[j + 1] : 0.0f;
        a.z = j + 2 < cols ? ar[j + 2] : 0.0f;
        a.w = j + 3 < cols ? ar[j + 3] : 0.0f;
      }
      lr[j4] = make_float4(tf32_rna(a.x - tf32_trunc(a.x)), tf32_rna(a.y - tf32_trunc(a.y)),
                           tf32_rna(a.z - tf32_trunc(a.z)), tf32_rna(a.w - tf32_trunc(a.w)));
    }
  }
}

// ----------------------------------------------------------------- host side
// rows x kp fp32, K-major; box = 32 (k) x box_rows
static int make_kmajor_map(CUtensorMap* map, const float* base, int64_t rows, int64_t kp,
                           uint32_t box_rows) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(LAPIS_B200_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {(cuuint64_t)kp, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)kp * sizeof(float)};
  const cuuint32_t box[2] = {(cuuint32_t)TG_BK, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(LAPIS_B200_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  return LAPIS_B200_OK;
}

// rows x cols fp32 row-major (pitch ld elements), box = box_inner x box_rows
static int make_rowmajor_map(CUtensorMap* map, const float* base, int64_t rows, int64_t cols,
                             int64_t ld, uint32_t box_inner, uint32_t box_rows,
                             CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(LAPIS_B200_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(float)};
  const cuuint32_t box[2] = {box_inner, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(LAPIS_B200_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  return LAPIS_B200_OK;
}

// raw-head path: A 16-byte aligned with a 16-byte row pitch.  (Reading B
// MN-major straight from the caller's row-major B — TMA 128-B / 32-B-atom
// swizzle, UMMA layout type 1 — was measured too: correct, but the kernel
// ran 0.633 vs 0.57 ms at 4096^3, more than the transpose it saves.)
static bool tf32_raw_ok(const void* A, int64_t lda, int64_t sA, int64_t batch) {
  static const int off = [] {
    const char* e = getenv("LAPIS_B200_TF32_RAW");
    return (e && e[0] == '0') ? 1 : 0;
  }();
  if (off) return false;
  return (uintptr_t)A % 16 == 0 && lda % 4 == 0 && (batch <= 1 || sA % 4 == 0);
}

int gemm_tf32x3(int64_t batch, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda,
                const void* B, int64_t ldb, void* C, int64_t ldc, int64_t sA, int64_t sB,
                int64_t sC, cudaStream_t st, Guard guard) {
  if (m > 0x7fffffff || n > 0x7fffffff || k > 0x7fffffff)
    return fail(LAPIS_B200_ERR_ARG, "gemm tf32x3: extent too large");
  const int64_t kp = (k + 3) / 4 * 4;  // 16-byte row pitch for TMA
  if (k == 0) {
    for (int64_t b = 0; b < batch; ++b)
      for (int64_t i = 0; i < m; ++i)
        LB_TRY(check_cuda(cudaMemsetAsync((float*)C + b * sC + i * ldc, 0, n * sizeof(float), st),
                          "memset C"));
    return LAPIS_B200_OK;
  }
  static thread_local int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    LB_TRY(check_cuda(cudaFuncSetAttribute(gemm_tf32x3_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TG_SMEM),
                      "smem attr (gemm_tf32x3_kernel)"));
    configured_dev = dev;
  }
  if (tf32_raw_ok(A, lda, sA, batch)) {
    // the head of A is A itself (read K-major straight from the caller's
    // row-major A); workspace: A's tail [m, kp], B's head and tail transposed
    float* ws = nullptr;
    const size_t a_elems = (size_t)m * kp, b_elems = (size_t)n * kp;
    LB_TRY(check_cuda(cudaMallocAsync((void**)&ws, (a_elems + 2 * b_elems) * sizeof(float), st),
                      "alloc(tf32x3 workspace)"));
    float* al = ws;
    float* bh = al + a_elems;
    float* bl = bh + b_elems;
    int rc = LAPIS_B200_OK;
    for (int64_t b = 0; b < batch && rc == LAPIS_B200_OK; ++b) {
      const float* Ab = (const float*)A + b * sA;
      const float* Bb = (const float*)B + b * sB;
      float* Cb = (float*)C + b * sC;
      const int64_t ga = std::min<int64_t>(m, (int64_t)num_sms() * 16);
      tf32_tail_kernel<<<(unsigned)ga, 256, 0, st>>>(m, k, kp, Ab, lda, al, guard);
      dim3 tg((unsigned)((n + 63) / 64), (unsigned)((kp + 63) / 64));
      split_transpose_kernel<<<tg, 256, 0, st>>>(k, n, kp, Bb, ldb, bh, bl, guard, 1);
      rc = check_launch("tf32 split (raw A head)");
      CUtensorMap mah, mal, mbh, mbl;
      if (rc == LAPIS_B200_OK) rc = make_rowmajor_map(&mah, Ab, m, k, lda, TG_BK, TG_BM);
      if (rc == LAPIS_B200_OK) rc = make_kmajor_map(&mal, al, m, kp, TG_BM);
      if (rc == LAPIS_B200_OK) rc = make_kmajor_map(&mbh, bh, n, kp, TG_BN);
      if (rc == LAPIS_B200_OK) rc = make_kmajor_map(&mbl, bl, n, kp, TG_BN);
      if (rc != LAPIS_B200_OK) break;
      Tf32Params prm;
      prm.m = (int)m;
      prm.n = (int)n;
      prm.nk = (int)((kp + TG_BK - 1) / TG_BK);
      prm.num_m = (int)((m + TG_BM - 1) / TG_BM);
      prm.num_n = (int)((n + TG_BN - 1) / TG_BN);
      prm.C = Cb;
      prm.ldc = ldc;
      const int tiles = prm.num_m * prm.num_n;
      const int grid = std::min(tiles, num_sms());
      gemm_tf32x3_kernel<<<grid, TG_THREADS_V2, TG_SMEM, st>>>(mah, mal, mbh, mbl, prm, guard);
      rc = check_launch("gemm_tf32x3_kernel");
    }
    cudaFreeAsync(ws, st);
    return rc;
  }
  float* ws = nullptr;
  const size_t a_elems = (size_t)m * kp, b_elems = (size_t)n * kp;
  LB_TRY(check_cuda(cudaMallocAsync((void**)&ws, 2 * (a_elems + b_elems) * sizeof(float), st),
                    "alloc(tf32x3 workspace)"));
  float* ah = ws;
  float* al = ah + a_elems;
  float* bh = al + a_elems;
  float* bl = bh + b_elems;
  int rc = LAPIS_B200_OK;
  for (int64_t b = 0; b < batch && rc == LAPIS_B200_OK; ++b) {
    const float* Ab = (const float*)A + b * sA;
    const float* Bb = (const float*)B + b * sB;
    float* Cb = (float*)C + b * sC;
    const int64_t sblocks = std::min<int64_t>(m, (int64_t)num_sms() * 16);
    static const int rawhi = [] {
      const char* e = getenv("LAPIS_B200_TF32_RAWHI");
      return (e && e[0] == '1') ? 1 : 0;
    }();
    split_rows_kernel<<<(unsigned)sblocks, 256, 0, st>>>(m, k, kp, Ab, lda, ah, al, guard, rawhi);
    dim3 tg((unsigned)((n + 63) / 64), (unsigned)((kp + 63) / 64));
    split_transpose_kernel<<<tg, 256, 0, st>>>(k, n, kp, Bb, ldb, bh, bl, guard, rawhi);
    rc = check_launch("tf32 split");
    CUtensorMap mah, mal, mbh, mbl;
    if (rc == LAPIS_B200_OK) rc = make_kmajor_map(&mah, ah, m, kp, TG_BM);
    if (rc == LAPIS_B200_OK) rc = make_kmajor_map(&mal, al, m, kp, TG_BM);
    if (rc == LAPIS_B200_OK) rc = make_kmajor_map(&mbh, bh, n, kp, TG_BN);
    if (rc == LAPIS_B200_OK) rc = make_kmajor_map(&mbl, bl, n, kp, TG_BN);
    if (rc != LAPIS_B200_OK) break;
    Tf32Params prm;
    prm.m = (int)m;
    prm.n = (int)n;
    prm.nk = (int)((kp + TG_BK - 1) / TG_BK);
    prm.num_m = (int)((m + TG_BM - 1) / TG_BM);
    prm.num_n = (int)((n + TG_BN - 1) / TG_BN);
    prm.C = Cb;
    prm.ldc = ldc;
    const int tiles = prm.num_m * prm.num_n;
    const int grid = std::min(tiles, num_sms());
    gemm_tf32x3_kernel<<<grid, TG_THREADS_V2, TG_SMEM, st>>>(mah, mal, mbh, mbl, prm, guard);
    rc = check_launch("gemm_tf32x3_kernel");
  }
  cudaFreeAsync(ws, st);
  return rc;
}

}  // namespace lapis_b200
