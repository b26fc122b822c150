// gemm_ozaki.cu — fp64 / fp32 dense matmul on the int8 tensor cores.
//
// C = A * B (row-major) for linalg.matmul / kokkos.gemm (interp.py:711-722,
// runtime_header.py:249-266) through the Ozaki splitting scheme: every row of
// A (column of B) is scaled by a power of two into (-1, 1) and cut into S
// signed 7-bit digits,
//     a_ij = 2^ea_i * sum_s  A_s[i,j] * 2^(-7(s+1)) + r,   |r| < 2^(ea_i - 7S),
// so that  C ~= 2^(ea_i + eb_j) * sum_{d<S} 2^(-7(d+2)) * C_d,
//          C_d = sum_{s+t=d} A_s B_t   (exact int32 products and sums).
// Each C_d is one int8 GEMM with a concatenated K' = (d+1) K on
// tcgen05.mma kind::i8 (UTCIMMA): S(S+1)/2 slice products in total.  S = 8 for
// fp64 (36 products; 6.8e-14 worst relative error at 4096^3 against the
// reference's sequential fp64 sum, contract 1e-12) and S = 4 for fp32 (10
// products; the reference's own fp32 rounding dominates).  SURVEY H2 "stretch:
// Ozaki fp64 emulation on kind::i8".
//
// Kernel shape (one CTA per SM, persistent over 128x256 output tiles), the
// warp roles of gemm_tf32x3.cu:
//   warp 0     TMA producer: 128x128 A-digit and 256x128 B-digit boxes (int8,
//              SWIZZLE_128B) into a 4-stage ring
//   warp 1     TMEM allocator + MMA issuer: M=128 N=256 K=32 int8 MMAs into a
//              double-buffered s32 accumulator (2 x 256 TMEM columns), one
//              accumulator per diagonal d
//   warps 2-9  epilogue: tcgen05.ld the s32 diagonal, scale by
//              2^(ea_i + eb_j - 7(d+2)) in fp64 and add it to the tile's fp64
//              partial (the output itself for fp64, a workspace for fp32,
//              L2-resident between diagonals); the last diagonal writes C.
// Non-finite inputs cannot be digit-split: the split kernels raise a device
// flag, the Ozaki kernel then returns at once and a guarded reference-order
// GEMM computes C instead (all stream-ordered, no host sync).
#include "common.cuh"
#include "tcgen05.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace lapis_b200 {

constexpr int OZ_BM = 128, OZ_BK = 128, OZ_STAGES = 4, OZ_UMMA_K = 32;
constexpr uint32_t OZ_A_BYTES = OZ_BM * OZ_BK;   // 16 KB
constexpr uint32_t OZ_TMEM_COLS = 512;
constexpr size_t OZ_EPI_SMEM = 8 * 32 * 16 * sizeof(double);   // per-warp transpose tiles
// tile N: 256 (fewer operand bytes per MMA) or 192 (finer tile grid); per dtype
template <int BN> struct OzTile {
  static constexpr int HALF = BN / 2;                       // columns per epilogue warp
  static constexpr uint32_t B_BYTES = BN * OZ_BK;
  static constexpr uint32_t STAGE_BYTES = OZ_A_BYTES + B_BYTES;
  static constexpr size_t SMEM = (size_t)OZ_STAGES * STAGE_BYTES + OZ_EPI_SMEM + 1024;
};
constexpr int OZ_EPI_WARPS = 8;
constexpr int OZ_THREADS = 64 + OZ_EPI_WARPS * 32;
constexpr int OZ_MAX_S = 9;

struct OzParams {
  int m, n, nk, num_m, num_n, S;
  int mp, np;               // slice row pitches (multiples of the tile)
  void* C;                  // OUT*
  int64_t ldc;
  double* part;             // fp64 partial sums (== C for fp64 output)
  int64_t ldp;
  const int* ea;            // [m] row exponents
  const int* eb;            // [n] column exponents
  int* flag;                // [0] non-finite input (skip), [1] certification failed
  double cert_k;            // error bound per unit 2^(ea+eb): K * per-product bound
  double cert_tol;          // certified |C - exact| <= cert_tol * max(|C|, 1)
  bool vec2;                // 16-byte partial accesses (even pitch, aligned)
  int sign_gate;            // 1: a negative operand entry (split kernels raise flag[1]) skips the kernel
  unsigned long long* prof; // optional: wait-cycle counters (LAPIS_B200_OZAKI_PROF=1)
  int digits8;              // 1: signed 8-bit leading digit + unsigned 8-bit digits
  // last-wave split (tiles >= split_base): the owner CTA runs the diagonals in
  // owner_mask (always the last one), a helper CTA the rest into its own fp64
  // tile in `split_ws` and raises one flag per epilogue warp; the owner adds
  // that tile before its last diagonal
  int split_base, nsplit;
  uint32_t owner_mask, helper_mask;
  double* split_ws;         // [nsplit][OZ_BM][BN]
  int* split_flag;          // [nsplit][OZ_EPI_WARPS], zeroed per call
};

// Work item k of this CTA: whole tiles blockIdx.x + k * gridDim.x below
// split_base (a multiple of gridDim.x), then at most one half of a split tile.
struct OzItem {
  int tile, role, slot;     // role 0 whole, 1 owner, 2 helper
  uint32_t mask;            // diagonals this item runs
};
__device__ __forceinline__ bool oz_item(const OzParams& p, int k, OzItem& it) {
  const int t = blockIdx.x + k * gridDim.x;
  if (t < p.split_base) {
    it.tile = t; it.role = 0; it.slot = 0; it.mask = (1u << p.S) - 1u;
    return true;
  }
  if (k * (int)gridDim.x != p.split_base || (int)blockIdx.x >= 2 * p.nsplit) return false;
  it.slot = blockIdx.x >> 1;
  it.tile = p.split_base + it.slot;
  it.role = 1 + (blockIdx.x & 1);
  it.mask = it.role == 1 ? p.owner_mask : p.helper_mask;
  return true;
}
__device__ __forceinline__ int ld_acquire(const int* ptr) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(ptr) : "memory");
  return v;
}

__device__ __forceinline__ void tc_mma_i8(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
      :: "r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// the same for a CTA pair (M = 256: rows 0-127 in the leader's TMEM, 128-255
// in the peer's; B's N split 64 + 64 between their shared memories); issued
// by the leader only
__device__ __forceinline__ void tc_mma_i8_2sm(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}"
      :: "r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// instruction descriptor: D s32 (2), A/B 8-bit signed (1) or unsigned (0),
// both K-major, N>>3, M>>4
__host__ __device__ constexpr uint32_t i8_idesc(int M, int N, bool a_signed = true,
                                                bool b_signed = true) {
  return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | ((b_signed ? 1u : 0u) << 10) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// x * 2^e for an integer-valued x (|x| < 2^53), correctly rounded like scalbn,
// branch-free: two multiplies by constructed powers of two, the first clamped
// to the normal range (exact for such x), the second carrying the rest (1.0
// for every in-range e).  Branch-free keeps the unrolled epilogues small enough
// for the instruction cache (an inlined scalbn per element does not fit).
__device__ __forceinline__ double pow2_scale(double x, int e) {
  const int e1 = min(max(e, -1022), 1023);
  const int e2 = min(max(e - e1, -1022), 1023);
  return x * __hiloint2double((e1 + 1023) << 20, 0) * __hiloint2double((e2 + 1023) << 20, 0);
}

// Drain one s32 diagonal of this warp's 32 x HALF accumulator slice: scale by
// 2^(shift + eb_j), add to the fp64 partial at pbase (the output / fp32
// workspace with pitch ldp, or a helper's tile with pitch OZ_BN) and, for the
// last diagonal, certify and write C.
template <class OUT, int OZ_BN, bool HELPER>
__device__ __forceinline__ void oz_drain(const OzParams& p, double* wsm, uint32_t tbase, int row_base,
                                         int col0, int shift, bool read_old, bool last,
                                         double* pbase) {
  const int lane = threadIdx.x & 31;
#pragma unroll 1
  for (int c0 = 0; c0 < OzTile<OZ_BN>::HALF; c0 += 16) {
    uint32_t v[16];
    tmem_ld_x16(tbase + (uint32_t)c0, v);
    const int cb = col0 + c0;
    // scale this thread's row segment, then transpose it through the
    // warp's shared tile (16-byte pairs XOR-swizzled by row) so that the
    // partial's read-modify-write is 4 rows x 128 B per instruction
#pragma unroll
    for (int pq = 0; pq < 8; ++pq) {
      const int q = 2 * pq;
      const int e0 = (cb + q < p.n) ? __ldg(p.eb + cb + q) : 0;
      const int e1 = (cb + q + 1 < p.n) ? __ldg(p.eb + cb + q + 1) : 0;
      const double x0 = pow2_scale((double)(int)v[q], shift + e0);
      const double x1 = pow2_scale((double)(int)v[q + 1], shift + e1);
      *reinterpret_cast<double2*>(wsm + lane * 16 + 2 * (pq ^ (lane & 7))) = make_double2(x0, x1);
    }
    __syncwarp();
    double2 t[8];
    const int pq = lane & 7;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = 4 * i + (lane >> 3);
      t[i] = *reinterpret_cast<const double2*>(wsm + r * 16 + 2 * (pq ^ (r & 7)));
    }
    __syncwarp();
    const int gc = cb + 2 * pq;
    double2 old[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int gr = row_base + 4 * i + (lane >> 3);
      old[i] = make_double2(0.0, 0.0);
      if (read_old && gr < p.m) {
        const double* src = pbase + (int64_t)gr * (HELPER ? OZ_BN : p.ldp) + gc;
        if (p.vec2 && gc + 1 < p.n) old[i] = *reinterpret_cast<const double2*>(src);
        else {
          if (gc < p.n) old[i].x = src[0];
          if (gc + 1 < p.n) old[i].y = src[1];
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int gr = row_base + 4 * i + (lane >> 3);
      if (gr >= p.m) continue;
      const double y0 = t[i].x + old[i].x, y1 = t[i].y + old[i].y;
      if (!HELPER && last) {
        // certify |y - exact| <= cert_tol * max(|y|, 1) from the a-priori bound
        const int er = __ldg(p.ea + gr);
        const double b0 = pow2_scale(p.cert_k, er + (gc < p.n ? __ldg(p.eb + gc) : 0));
        const double b1 = pow2_scale(p.cert_k, er + (gc + 1 < p.n ? __ldg(p.eb + gc + 1) : 0));
        if ((gc < p.n && b0 > p.cert_tol * fmax(fabs(y0), 1.0)) ||
            (gc + 1 < p.n && b1 > p.cert_tol * fmax(fabs(y1), 1.0)))
          atomicExch(p.flag + 1, 1);
        OUT* dst = reinterpret_cast<OUT*>(p.C) + (int64_t)gr * p.ldc + gc;
        if (gc < p.n) dst[0] = (OUT)y0;
        if (gc + 1 < p.n) dst[1] = (OUT)y1;
      } else {
        double* dst = pbase + (int64_t)gr * (HELPER ? OZ_BN : p.ldp) + gc;
        if (p.vec2 && gc + 1 < p.n) *reinterpret_cast<double2*>(dst) = make_double2(y0, y1);
        else {
          if (gc < p.n) dst[0] = y0;
          if (gc + 1 < p.n) dst[1] = y1;
        }
      }
    }
  }
}

template <class OUT, int OZ_BN>
__global__ void __launch_bounds__(OZ_THREADS, 1)
gemm_ozaki_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                  OzParams p) {
  if (p.flag[0] || (p.sign_gate && p.flag[1])) return;  // uniform: a guarded fallback owns this call
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[OZ_STAGES], empty[OZ_STAGES], tmem_full[2], tmem_empty[2];
  __shared__ uint32_t tmem_base_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = p.S;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tA);
    prefetch_tmap(&tB);
    for (int s = 0; s < OZ_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], OZ_EPI_WARPS * 32);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(&tmem_base_slot)), "r"(OZ_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ producer
      int stage = 0;
      uint32_t phase = 0;
      long long prod_wait = 0;
      OzItem it;
      for (int k = 0; oz_item(p, k, it); ++k) {
        const int mb = it.tile % p.num_m, nb = it.tile / p.num_m;
        for (int d = 0; d < S; ++d)
          if ((it.mask >> d) & 1u)
          for (int s = 0; s <= d; ++s)
            for (int kb = 0; kb < p.nk; ++kb) {
              const long long t0 = p.prof ? clock64() : 0;
              mbar_wait(&empty[stage], phase ^ 1);
              if (p.prof) prod_wait += clock64() - t0;
              uint8_t* sa = smem + stage * OzTile<OZ_BN>::STAGE_BYTES;
              mbar_arrive_expect_tx(&full[stage], OzTile<OZ_BN>::STAGE_BYTES);
              tma_load_2d(sa, &tA, kb * OZ_BK, s * p.mp + mb * OZ_BM, &full[stage]);
              tma_load_2d(sa + OZ_A_BYTES, &tB, kb * OZ_BK, (d - s) * p.np + nb * OZ_BN, &full[stage]);
              if (++stage == OZ_STAGES) { stage = 0; phase ^= 1; }
            }
      }
      if (p.prof) atomicAdd(p.prof + 0, (unsigned long long)prod_wait);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------------------------------------------------- MMA issuer
      // 7-bit digits: all signed.  8-bit digits: only digit 0 is signed.
      constexpr uint32_t idesc_ss = i8_idesc(OZ_BM, OZ_BN, true, true);
      constexpr uint32_t idesc_su = i8_idesc(OZ_BM, OZ_BN, true, false);
      constexpr uint32_t idesc_us = i8_idesc(OZ_BM, OZ_BN, false, true);
      constexpr uint32_t idesc_uu = i8_idesc(OZ_BM, OZ_BN, false, false);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      long long w_tmem = 0, w_full = 0;
      const long long t_start = clock64();
      OzItem it;
      for (int k = 0; oz_item(p, k, it); ++k) {
        for (int d = 0; d < S; ++d) {
          if (!((it.mask >> d) & 1u)) continue;
          long long t0 = p.prof ? clock64() : 0;
          mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
          if (p.prof) w_tmem += clock64() - t0;
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + (uint32_t)(acc * OZ_BN);
          bool first = true;
          for (int s = 0; s <= d; ++s) {
            const uint32_t idesc = !p.digits8 ? idesc_ss
                                 : (s == 0 ? (d == 0 ? idesc_ss : idesc_su)
                                           : (d - s == 0 ? idesc_us : idesc_uu));
            for (int kb = 0; kb < p.nk; ++kb) {
              t0 = p.prof ? clock64() : 0;
              mbar_wait(&full[stage], phase);
              if (p.prof) w_full += clock64() - t0;
              tc_fence_after();
              const uint8_t* sa = smem + stage * OzTile<OZ_BN>::STAGE_BYTES;
              const uint64_t adesc = smem_desc_sw128(sa);
              const uint64_t bdesc = smem_desc_sw128(sa + OZ_A_BYTES);
#pragma unroll
              for (int kk = 0; kk < OZ_BK / OZ_UMMA_K; ++kk) {
                // 32 bytes of K per MMA: advance the start address inside the swizzle atom
                tc_mma_i8(d_tmem, adesc + (uint64_t)(kk * 2), bdesc + (uint64_t)(kk * 2), idesc,
                          first ? 0u : 1u);
                first = false;
              }
              tc_commit(&empty[stage]);
              if (++stage == OZ_STAGES) { stage = 0; phase ^= 1; }
            }
          }
          tc_commit(&tmem_full[acc]);
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
      }
      if (p.prof) {
        atomicAdd(p.prof + 1, (unsigned long long)w_tmem);
        atomicAdd(p.prof + 2, (unsigned long long)w_full);
        atomicAdd(p.prof + 3, (unsigned long long)(clock64() - t_start));
      }
    }
  } else {
    // ------------------------------------------------------------- epilogue
    const int ew = warp - 2;                 // 0..7
    double* wsm = reinterpret_cast<double*>(smem + OZ_STAGES * OzTile<OZ_BN>::STAGE_BYTES) + ew * 32 * 16;
    const int lg = warp & 3;                 // TMEM lane group this warp may access
    const int half = ew >> 2;                // columns [128*half, 128*half + 128)
    int acc = 0;
    uint32_t acc_phase = 0;
    OzItem it;
    for (int k = 0; oz_item(p, k, it); ++k) {
      const int mb = it.tile % p.num_m, nb = it.tile / p.num_m;
      const int row_base = mb * OZ_BM + lg * 32;
      // a helper accumulates into its own tile (pitch OZ_BN), indexed by the
      // output's row / column
      double* const hbase = p.split_ws + (int64_t)it.slot * OZ_BM * OZ_BN -
                            (int64_t)mb * OZ_BM * OZ_BN - nb * OZ_BN;
      const int d_first = __ffs(it.mask) - 1, d_last = 31 - __clz(it.mask);
      const int row = row_base + lane;
      const int col0 = nb * OZ_BN + half * OzTile<OZ_BN>::HALF;
      const int ea = row < p.m ? p.ea[row] : 0;
      for (int d = 0; d < S; ++d) {
        if (!((it.mask >> d) & 1u)) continue;
        const long long t0 = (p.prof && threadIdx.x == 64) ? clock64() : 0;
        mbar_wait(&tmem_full[acc], acc_phase);
        if (p.prof && threadIdx.x == 64) atomicAdd(p.prof + 4, (unsigned long long)(clock64() - t0));
        tc_fence_after();
        const uint32_t tbase = tmem_base + ((uint32_t)(lg * 32) << 16) +
                               (uint32_t)(acc * OZ_BN + half * OzTile<OZ_BN>::HALF);
        const int shift = p.digits8 ? ea - 14 - 8 * d : ea - 7 * (d + 2);
        const bool last = d == d_last && it.role != 2;
        if (last && it.role == 1) {
          // owner: add the helper's tile into the partial first (a plain pass;
          // it is the only partial when the owner runs a single diagonal)
          const int* f = p.split_flag + it.slot * OZ_EPI_WARPS + ew;
          while (ld_acquire(f) == 0) __nanosleep(128);   // every lane acquires
          const double* hws = p.split_ws + (int64_t)it.slot * OZ_BM * OZ_BN + (lg * 32) * OZ_BN +
                              half * OzTile<OZ_BN>::HALF;
          for (int r = 0; r < 32; ++r) {
            const int gr = row_base + r;
            if (gr >= p.m) break;
            for (int c = lane; c < OzTile<OZ_BN>::HALF; c += 32) {
              const int gc = col0 + c;
              if (gc < p.n) {
                double* dst = p.part + (int64_t)gr * p.ldp + gc;
                *dst = (d == d_first ? 0.0 : *dst) + hws[r * OZ_BN + c];
              }
            }
          }
          __syncwarp();
        }
        const bool read_old = d != d_first || (last && it.role == 1);
        const long long t1 = (p.prof && threadIdx.x == 64) ? clock64() : 0;
        if (it.role == 2)
          oz_drain<OUT, OZ_BN, true>(p, wsm, tbase, row_base, col0, shift, read_old, false, hbase);
        else
          oz_drain<OUT, OZ_BN, false>(p, wsm, tbase, row_base, col0, shift, read_old, last, p.part);
        if (p.prof && threadIdx.x == 64) {
          atomicAdd(p.prof + 5, (unsigned long long)(clock64() - t1));
          atomicAdd(p.prof + 6, 1ull);
        }
        tc_fence_before();
        mbar_arrive(&tmem_empty[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        if (it.role == 2 && d == d_last) {
          // publish this warp's rows of the helper tile to the owner
          __threadfence();
          __syncwarp();
          if (lane == 0) atomicAdd(p.split_flag + it.slot * OZ_EPI_WARPS + ew, 1);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;"
                 :: "r"(tmem_base), "r"(OZ_TMEM_COLS));
  }
}

// ------------------------------------------------------- two-pass kernel
// fp64, S = 8: the diagonals' s32 accumulators live in TMEM four at a time
// (4 x 128 columns), so each K block's digit tiles are loaded ONCE and feed
// every slice product of a pass:
//   pass A  diagonals 0-3: digits 0-3 of A and B, 10 products per K block
//   pass B  diagonals 4-7: digits 0-7,            26 products per K block
// against S(S+1)/2 = 36 re-streamed tile pairs per K block in the
// per-diagonal kernel above, whose operand stream is L2->SM bound.  A stage
// is 64 KB: two K blocks of 4+4 digit tiles (pass A) or one K block of 8+8
// (pass B), each digit tile 128 x 32 int8 (SWIZZLE_32B, one 3-D TMA box per
// 4 digits).  The epilogue folds pass A's diagonals into an fp64 partial kept
// in a per-CTA L2-resident slot, then adds pass B's in ascending d — the
// per-diagonal kernel's summation order, so both kernels give identical bits.
constexpr int OZ2_BN = 128, OZ2_BK = 32, OZ2_STAGES = 3;
constexpr uint32_t OZ2_DIGIT = 128 * OZ2_BK;                 // 4 KB
constexpr uint32_t OZ2_STAGE = 16 * OZ2_DIGIT;               // 64 KB
constexpr size_t OZ2_SMEM = (size_t)OZ2_STAGES * OZ2_STAGE + OZ_EPI_SMEM + 1024;
constexpr int OZ2_SLOT = 8 * 4 * 16 * 32;                    // doubles per CTA partial (128 KB)

// Grouped raster: bands of OZ2_GM row blocks, column-major inside a band, so
// the ~148 tiles in flight share ~12 A and ~12 B digit blocks (instead of all
// 32 A blocks) and the concurrent CTAs hit the same lines in L2
#ifndef OZ2_GM
#define OZ2_GM 12
#endif
__device__ __forceinline__ void oz2_tile(int tile, int num_m, int num_n, int& mb, int& nb) {
  const int band = OZ2_GM * num_n;
  const int first = (tile / band) * OZ2_GM;
  const int rows = min(num_m - first, OZ2_GM);
  const int t = tile % band;
  mb = first + t % rows;
  nb = t / rows;
}

// NPASS = 2, SD = 8 (fp64, 7-bit signed digits) as described above; NPASS = 1,
// SD = 3, D8 (fp32, 8-bit digits: signed leading, unsigned others): pass A
// alone covers all 3 diagonals (6 products per K block) — the K blocks'
// digit tiles are streamed once, against 1 + 2 + 3 re-streamed K passes in
// the per-diagonal kernel.
// CM x CN clusters: the cluster takes CM row blocks x CN column blocks at a
// time; the CTAs of one row block share its A digit boxes and those of one
// column block its B digit boxes — each such box is loaded by ONE CTA and
// multicast into its sharers' shared memory (the operand stream from L2
// shrinks by the sharing factor).  A stage is refilled once every CTA that
// writes into it saw it released: each CTA's MMA commit is multicast to
// itself, its row peer and its column peer, and the empty barriers count
// 1 + (CN > 1) + (CM > 1) commits.
// P2 (CM = 2, CN = 1): the pair runs cta_group::2 MMAs, M = 256 — each CTA
// stages its own 128 A rows and 64 of the tile's 128 B rows (tB's box is 64
// rows), both CTAs' boxes complete on the leader's full barrier, the leader
// alone issues the MMAs and its commits release both CTAs' stages and
// accumulators; each CTA drains its own TMEM half.  Per dispatch an SM reads
// 4 KB of A + 2 KB of B from shared memory instead of 4 + 4 KB.
template <class OUT, int NPASS = 2, int SD = 8, bool D8 = false, int CM = 1, int CN = 1,
          bool P2 = false>
__global__ void __launch_bounds__(OZ_THREADS, 1)
gemm_ozaki_2p_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                     OzParams p) {
  static_assert((NPASS == 2 && SD == 8) || (NPASS == 1 && SD <= 4), "pass layout");
  constexpr int DA = SD < 4 ? SD : 4;   // diagonals of pass A
  // stage layout: pass A holds 2 K blocks of SL A digit tiles + SL B digit
  // tiles; one pass (SL = DA digits, 48 KB stages for fp32) fits NST = 4 stages
  // in the space of the two-pass kernel's three 64 KB stages
  constexpr int SL = NPASS == 1 ? DA : 4;
  // (P2: a CTA stages half of each B digit plane, so its stages are 3/4 the
  // size and one more fits — the pair's MMAs outrun three stages of TMA)
  constexpr uint32_t BD = P2 ? OZ2_DIGIT / 2 : OZ2_DIGIT;   // bytes per staged B digit plane
  constexpr uint32_t HB = SL * (OZ2_DIGIT + BD);             // pass-A half stage: SL A + SL B planes
  constexpr uint32_t STG = NPASS == 1 ? 2u * HB : 8u * (OZ2_DIGIT + BD);
  constexpr int NST = (int)((OZ2_STAGES * OZ2_STAGE) / STG);
  if (p.flag[0] || (p.sign_gate && p.flag[1])) return;  // uniform: a guarded fallback owns this call
  constexpr bool CL = CM * CN > 1;
  static_assert((CM == 1 || CM == 2) && (CN == 1 || CN == 2), "cluster shape");
  const uint32_t crank = CL ? cluster_ctarank() : 0u;
  const int cm = (int)crank % CM, cn = (int)crank / CM;         // rank = cn * CM + cm
  // A boxes go to the CTAs of this row block (same cm), B boxes to those of
  // this column block (same cn); commits to self, row peer and column peer
  const uint16_t a_mask = (uint16_t)(CN == 2 ? ((1u << cm) | (1u << (CM + cm))) : (1u << crank));
  const uint16_t b_mask = (uint16_t)(CM == 2 ? ((1u << (cn * CM)) | (1u << (cn * CM + 1))) : (1u << crank));
  const uint16_t c_mask = (uint16_t)(a_mask | b_mask);
  static_assert(!P2 || (CM == 2 && CN == 1), "CTA pairs along m");
  const bool leader = !P2 || crank == 0;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[NST], empty[NST], acc_full, acc_empty;
  __shared__ uint32_t tmem_base_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = p.nk, nk2 = (p.nk + 1) / 2;
  // work units: CM x CN groups of tiles, one per cluster at a time
  const int units = (p.num_m / CM) * (p.num_n / CN);
  const int ustart = (int)blockIdx.x / (CM * CN);
  const int ustride = (int)gridDim.x / (CM * CN);
  auto unit_tile = [&](int u, int& mb, int& nb) {
    int mg, ng;
    oz2_tile(u, p.num_m / CM, p.num_n / CN, mg, ng);
    mb = mg * CM + cm;
    nb = ng * CN + cn;
  };

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tA);
    prefetch_tmap(&tB);
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], P2 ? 1 : 1 + (CN > 1 ? 1 : 0) + (CM > 1 ? 1 : 0));
    }
    mbar_init(&acc_full, 1);
    mbar_init(&acc_empty, (P2 ? 2 : 1) * OZ_EPI_WARPS * 32);
    fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (P2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                   :: "r"(smem_u32(&tmem_base_slot)), "r"(OZ_TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                   :: "r"(smem_u32(&tmem_base_slot)), "r"(OZ_TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if constexpr (CL) cluster_sync_all();   // the peer's barriers exist before any multicast
  const uint32_t tmem_base = tmem_base_slot;
  const uint32_t full_cl0 = P2 ? smem_map_rank(&full[0], 0) : 0u;   // the leader's full barriers

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ producer
      int stage = 0;
      uint32_t phase = 0;
      // box b of a stage: shared boxes are loaded by the sharer whose index
      // in the sharing pair equals b % 2, multicast to both
      auto load_a = [&](void* dst, int kx, int ma, int dz, int b) {
        if constexpr (P2) {
          tma_load_3d_2sm(dst, &tA, kx, ma, dz, full_cl0 + 8u * stage);
        } else if constexpr (CN == 2) {
          if ((b & 1) == cn) tma_load_3d_mc(dst, &tA, kx, ma, dz, &full[stage], a_mask);
        } else {
          tma_load_3d(dst, &tA, kx, ma, dz, &full[stage]);
        }
      };
      auto load_b = [&](void* dst, int kx, int nbn, int dz, int b) {
        if constexpr (P2) {
          tma_load_3d_2sm(dst, &tB, kx, nbn + cm * 64, dz, full_cl0 + 8u * stage);
        } else if constexpr (CM == 2) {
          if ((b & 1) == cm) tma_load_3d_mc(dst, &tB, kx, nbn, dz, &full[stage], b_mask);
        } else {
          tma_load_3d(dst, &tB, kx, nbn, dz, &full[stage]);
        }
      };
      for (int u = ustart; u < units; u += ustride) {
        int mb, nb;
        unit_tile(u, mb, nb);
        const int ma = mb * OZ_BM, nbn = nb * OZ2_BN;
        for (int j = 0; j < nk2; ++j) {            // pass A: K blocks 2j, 2j+1 (zero-filled past K)
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STG;
          // boxes of DA digits (the 3-digit fp32 split loads no zero plane)
          if constexpr (P2) {
            if (leader) mbar_arrive_expect_tx(&full[stage], 2u * 2u * DA * (OZ2_DIGIT + BD));
          } else {
            mbar_arrive_expect_tx(&full[stage], 2u * 2u * DA * OZ2_DIGIT);
          }
          for (int h = 0; h < 2; ++h) {
            load_a(sa + h * HB, (2 * j + h) * OZ2_BK, ma, 0, h);
            load_b(sa + h * HB + SL * OZ2_DIGIT, (2 * j + h) * OZ2_BK, nbn, 0, h);
          }
          if (++stage == NST) { stage = 0; phase ^= 1; }
        }
        for (int kb = 0; kb < (NPASS == 2 ? nk : 0); ++kb) {   // pass B: one K block, all 8 digits
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STG;
          if constexpr (P2) {
            if (leader) mbar_arrive_expect_tx(&full[stage], 2u * 8u * (OZ2_DIGIT + BD));
          } else {
            mbar_arrive_expect_tx(&full[stage], OZ2_STAGE);
          }
          load_a(sa, kb * OZ2_BK, ma, 0, 0);
          load_a(sa + 4 * OZ2_DIGIT, kb * OZ2_BK, ma, 4, 1);
          load_b(sa + 8 * OZ2_DIGIT, kb * OZ2_BK, nbn, 0, 0);
          load_b(sa + 8 * OZ2_DIGIT + 4 * BD, kb * OZ2_BK, nbn, 4, 1);
          if (++stage == NST) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1 && leader) {
    // ------------------------------------------------------------ MMA issuer
    // (the whole warp runs the loop, one elected lane issues; P2: the leader's)
    constexpr int MM = P2 ? 2 * OZ_BM : OZ_BM;
    constexpr uint32_t idesc = i8_idesc(MM, OZ2_BN, true, true);
    // 8-bit digits: digit 0 signed, the others unsigned
    constexpr uint32_t idesc_su = i8_idesc(MM, OZ2_BN, true, false);
    constexpr uint32_t idesc_us = i8_idesc(MM, OZ2_BN, false, true);
    constexpr uint32_t idesc_uu = i8_idesc(MM, OZ2_BN, false, false);
    auto mma = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
      if constexpr (P2) tc_mma_i8_2sm(d, a, b, id, acc);
      else tc_mma_i8(d, a, b, id, acc);
    };
    int stage = 0;
    uint32_t phase = 0, acc_phase = 0;
    long long w_tmem = 0, w_full = 0;
    const long long t_start = clock64();
    for (int u = ustart; u < units; u += ustride) {
      for (int pass = 0; pass < NPASS; ++pass) {
        long long t0 = p.prof ? clock64() : 0;
        mbar_wait(&acc_empty, acc_phase ^ 1);
        if (p.prof) w_tmem += clock64() - t0;
        acc_phase ^= 1;
        tc_fence_after();
        const int nstage = pass == 0 ? nk2 : nk;
        for (int j = 0; j < nstage; ++j) {
          t0 = p.prof ? clock64() : 0;
          mbar_wait(&full[stage], phase);
          if (p.prof) w_full += clock64() - t0;
          tc_fence_after();
          const uint64_t desc0 = smem_desc_sw32(smem + stage * STG);
          if (elect_one()) {
            if (pass == 0) {
#pragma unroll
              for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int d = 0; d < DA; ++d)
#pragma unroll
                  for (int s = 0; s <= d; ++s)
                    mma(tmem_base + (uint32_t)(d * OZ2_BN),
                              desc0 + (uint64_t)((h * HB + s * OZ2_DIGIT) >> 4),
                              desc0 + (uint64_t)((h * HB + SL * OZ2_DIGIT + (d - s) * BD) >> 4),
                              !D8 ? idesc : (s == 0 ? (d == 0 ? idesc : idesc_su)
                                                    : (d - s == 0 ? idesc_us : idesc_uu)),
                              (j > 0 || h > 0 || s > 0) ? 1u : 0u);
            } else {
#pragma unroll
              for (int d = 4; d < 8; ++d)
#pragma unroll
                for (int s = 0; s <= d; ++s)
                  mma(tmem_base + (uint32_t)((d - 4) * OZ2_BN),
                            desc0 + (uint64_t)((s * OZ2_DIGIT) >> 4),
                            desc0 + (uint64_t)((8 * OZ2_DIGIT + (d - s) * BD) >> 4), idesc,
                            (j > 0 || s > 0) ? 1u : 0u);
            }
            if constexpr (P2) tc_commit_2sm_mc(&empty[stage], (uint16_t)3);
            else if constexpr (CL) tc_commit_mc(&empty[stage], c_mask);
            else tc_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == NST) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) {
          if constexpr (P2) tc_commit_2sm_mc(&acc_full, (uint16_t)3);
          else tc_commit(&acc_full);
        }
        __syncwarp();
      }
    }
    if (p.prof && lane == 0) {
      atomicAdd(p.prof + 1, (unsigned long long)w_tmem);
      atomicAdd(p.prof + 2, (unsigned long long)w_full);
      atomicAdd(p.prof + 3, (unsigned long long)(clock64() - t_start));
    }
  } else if (warp >= 2) {
    // ------------------------------------------------------------- epilogue
    const int ew = warp - 2;                 // 0..7
    const int lg = warp & 3;                 // TMEM lane group this warp may access
    const int half = ew >> 2;                // columns [64*half, 64*half + 64)
    double* wsm = reinterpret_cast<double*>(smem + OZ2_STAGES * OZ2_STAGE) + ew * 32 * 16;  // after the stages
    // this warp's partial in the CTA's slot: [chunk][j][lane], coalesced per j
    double* slot = p.split_ws + (int64_t)blockIdx.x * OZ2_SLOT + ew * (4 * 16 * 32) + lane;
    uint32_t acc_phase = 0;
    for (int u = ustart; u < units; u += ustride) {
      int mb, nb;
      unit_tile(u, mb, nb);
      const int row_base = mb * OZ_BM + lg * 32;
      const int row = row_base + lane;
      const int ea = row < p.m ? __ldg(p.ea + row) : 0;
      const uint32_t tbase = tmem_base + ((uint32_t)(lg * 32) << 16) + (uint32_t)(half * 64);
      for (int pass = 0; pass < NPASS; ++pass) {
        mbar_wait(&acc_full, acc_phase);
        acc_phase ^= 1;
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          const int cb = nb * OZ2_BN + half * 64 + c * 16;
          int e[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) e[j] = (cb + j < p.n) ? __ldg(p.eb + cb + j) : 0;
          double y[16];
          if (pass == 1) {
#pragma unroll
            for (int j = 0; j < 16; ++j) y[j] = slot[(c * 16 + j) * 32];
          }
          // the pass's diagonals combined exactly in 64-bit integers before
          // ONE conversion and scaling per element: t = sum_q v_q 2^(W (QN-1-q))
          // (|v_q| < 2^31, so |t| < 2^53: exact in int64 and in the
          // conversion); the per-diagonal double conversions, scalings and
          // adds were the drain's cost (the MMA thread waited on it 10 % of
          // its time)
          constexpr int W = D8 ? 8 : 7;
          const int qn = pass == 0 ? DA : 4;
          long long t[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) t[j] = 0;
#pragma unroll 1
          for (int q = 0; q < qn; ++q) {
            uint32_t v[16];
            tmem_ld_x16(tbase + (uint32_t)(q * OZ2_BN + c * 16), v);
#pragma unroll
            for (int j = 0; j < 16; ++j) t[j] = t[j] * (1ll << W) + (long long)(int)v[j];
          }
          const int dl = pass * 4 + qn - 1;   // the last diagonal sets the scale
          const int shift = D8 ? ea - 14 - 8 * dl : ea - 7 * (dl + 2);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const double x = pow2_scale((double)t[j], shift + e[j]);
            y[j] = pass == 0 ? x : x + y[j];
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) slot[(c * 16 + j) * 32] = y[j];
        }
        // every accumulator read: the next pass's MMAs may start
        tc_fence_before();
        if constexpr (P2) mbar_arrive_cl(smem_map_rank(&acc_empty, 0));
        else mbar_arrive(&acc_empty);
      }
      // final: certify and write C through the shared transpose (4 rows x 16
      // columns per store instruction)
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        const int cb = nb * OZ2_BN + half * 64 + c * 16;
        bool bad = false;
#pragma unroll
        for (int pq = 0; pq < 8; ++pq) {
          const double y0 = slot[(c * 16 + 2 * pq) * 32], y1 = slot[(c * 16 + 2 * pq + 1) * 32];
          const int c0 = cb + 2 * pq;
          if (row < p.m) {
            bad |= c0 < p.n && pow2_scale(p.cert_k, ea + __ldg(p.eb + c0)) > p.cert_tol * fmax(fabs(y0), 1.0);
            bad |= c0 + 1 < p.n &&
                   pow2_scale(p.cert_k, ea + __ldg(p.eb + c0 + 1)) > p.cert_tol * fmax(fabs(y1), 1.0);
          }
          *reinterpret_cast<double2*>(wsm + lane * 16 + 2 * (pq ^ (lane & 7))) = make_double2(y0, y1);
        }
        if (bad) atomicExch(p.flag + 1, 1);
        __syncwarp();
        const int pq = lane & 7;
        const int gc = cb + 2 * pq;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = 4 * i + (lane >> 3);
          const double2 t = *reinterpret_cast<const double2*>(wsm + r * 16 + 2 * (pq ^ (r & 7)));
          const int gr = row_base + r;
          if (gr >= p.m) continue;
          OUT* dst = reinterpret_cast<OUT*>(p.C) + (int64_t)gr * p.ldc + gc;
          if (p.vec2 && gc + 1 < p.n) {
            if constexpr (sizeof(OUT) == 8)
              *reinterpret_cast<double2*>(dst) = t;
            else
              *reinterpret_cast<float2*>(dst) = make_float2((float)t.x, (float)t.y);
          } else {
            if (gc < p.n) dst[0] = (OUT)t.x;
            if (gc + 1 < p.n) dst[1] = (OUT)t.y;
          }
        }
        __syncwarp();
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  // (CL) no CTA leaves while its peer may still multicast into it or arrive
  // on its barriers
  if constexpr (CL) cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (P2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;"
                   :: "r"(tmem_base), "r"(OZ_TMEM_COLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;"
                   :: "r"(tmem_base), "r"(OZ_TMEM_COLS));
  }
}

// ------------------------------------------------------------- digit split
// Peel the S signed 7-bit digits of r in (-1, 1) for 4 consecutive elements
// and store them as one 32-bit word per plane.  Sequential peeling
// (t = 128 r, digit = trunc(t), r = t - digit, all exact in fp64) yields the
// base-128 digits of trunc(|r| 2^(7S)) with r's sign, so one conversion per
// element replaces S of them.
__device__ __forceinline__ void peel4(double r0, double r1, double r2, double r3, int S,
                                      int8_t* __restrict__ out, int64_t plane) {
  const double r[4] = {r0, r1, r2, r3};
  const double scale = __hiloint2double((7 * S + 1023) << 20, 0);
  unsigned long long q[4];
  uint32_t neg = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    q[c] = (unsigned long long)(fabs(r[c]) * scale);   // exact scaling, truncating conversion
    neg |= (r[c] < 0.0 ? 1u : 0u) << c;
  }
  for (int s = 0; s < S; ++s) {
    const int sh = 7 * (S - 1 - s);
    uint32_t w = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int d = (int)((q[c] >> sh) & 127u);
      w |= (uint32_t)(uint8_t)((neg >> c) & 1u ? -d : d) << (8 * c);
    }
    *reinterpret_cast<uint32_t*>(out + (int64_t)s * plane) = w;
  }
}

// peel4 for S <= 8 without 64-bit integers: trunc(|r| 2^(7S)) is taken in
// two exact fp64 steps, a = |r| 2^28 (digits 0-3 from trunc(a)) and
// frac(a) 2^(7(S-4)) (digits 4..S-1), each converted to int32 — the same
// digits as peel4
__device__ __forceinline__ void peel4_fast(double r0, double r1, double r2, double r3, int S,
                                           int8_t* __restrict__ out, int64_t plane) {
  const double r[4] = {r0, r1, r2, r3};
  const int sh_hi = S < 4 ? 7 * S : 28;
  const double s_hi = __hiloint2double((sh_hi + 1023) << 20, 0);
  const double s_lo = __hiloint2double((7 * (S > 4 ? S - 4 : 0) + 1023) << 20, 0);
  uint32_t hi[4], lo[4];
  uint32_t neg = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double a = fabs(r[c]) * s_hi;
    const double t = trunc(a);
    hi[c] = (uint32_t)__double2uint_rz(t);
    lo[c] = (uint32_t)__double2uint_rz((a - t) * s_lo);
    neg |= (r[c] < 0.0 ? 1u : 0u) << c;
  }
  uint32_t* o = reinterpret_cast<uint32_t*>(out);
  const int64_t plane4 = plane >> 2;
  const int nhi = S < 4 ? S : 4;
  for (int s = 0; s < nhi; ++s) {
    const int sh = 7 * (nhi - 1 - s);
    uint32_t w = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint32_t d = (hi[c] >> sh) & 127u;
      w |= (uint32_t)(uint8_t)((neg >> c) & 1u ? (uint32_t)(-(int)d) : d) << (8 * c);
    }
    o[s * plane4] = w;
  }
  for (int s = 4; s < S; ++s) {
    const int sh = 7 * (S - 1 - s);
    uint32_t w = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint32_t d = (lo[c] >> sh) & 127u;
      w |= (uint32_t)(uint8_t)((neg >> c) & 1u ? (uint32_t)(-(int)d) : d) << (8 * c);
    }
    o[s * plane4] = w;
  }
}

// S = 8 (the fp64 default), fully unrolled: per plane the four 7-bit
// magnitudes are packed into one word with constant shifts, then negated as
// bytes at once for the negative elements — -b (mod 256) = (0x80 - b) ^ 0x80
// for 0 <= b <= 127, borrow-free across bytes — and selected by a byte mask
__device__ __forceinline__ void peel4_s8(double r0, double r1, double r2, double r3,
                                         int8_t* __restrict__ out, int64_t plane) {
  const double r[4] = {r0, r1, r2, r3};
  const double s28 = __hiloint2double((28 + 1023) << 20, 0);
  uint32_t hi[4], lo[4];
  uint32_t m = 0;   // 0xff in the bytes of negative elements
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double a = fabs(r[c]) * s28;
    const double t = trunc(a);
    hi[c] = __double2uint_rz(t);
    lo[c] = __double2uint_rz((a - t) * s28);
    m |= (r[c] < 0.0 ? 0xffu : 0u) << (8 * c);
  }
  uint32_t* o = reinterpret_cast<uint32_t*>(out);
  const int64_t p4 = plane >> 2;
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const uint32_t* q = s < 4 ? hi : lo;
    const int sh = 7 * (3 - (s & 3));
    const uint32_t w = ((q[0] >> sh) & 127u) | (((q[1] >> sh) & 127u) << 8) |
                       (((q[2] >> sh) & 127u) << 16) | (((q[3] >> sh) & 127u) << 24);
    const uint32_t wn = (0x80808080u - w) ^ 0x80808080u;
    o[s * p4] = (w & ~m) | (wn & m);
  }
}

// 8-bit digits: the leading digit floor(128 r) is signed ([-128, 127]), the
// remainder is in [0, 1) and every further digit floor(256 r) unsigned — the
// two's-complement bytes of floor(r 2^(7 + 8(S-1))).
__device__ __forceinline__ void peel4_u8(double r0, double r1, double r2, double r3, int S,
                                         int8_t* __restrict__ out, int64_t plane) {
  const double r[4] = {r0, r1, r2, r3};
  const double scale = __hiloint2double((7 + 8 * (S - 1) + 1023) << 20, 0);
  if (S <= 3) {   // |q| < 2^23: one rounding-down conversion to int32 per element
    int qi[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) qi[c] = __double2int_rd(r[c] * scale);
    for (int s = 0; s < S; ++s) {
      const int sh = 8 * (S - 1 - s);
      uint32_t w = 0;
#pragma unroll
      for (int c = 0; c < 4; ++c) w |= (uint32_t)((qi[c] >> sh) & 0xff) << (8 * c);
      *reinterpret_cast<uint32_t*>(out + (int64_t)s * plane) = w;
    }
    return;
  }
  long long q[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) q[c] = (long long)floor(r[c] * scale);
  for (int s = 0; s < S; ++s) {
    const int sh = 8 * (S - 1 - s);
    uint32_t w = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) w |= (uint32_t)((q[c] >> sh) & 0xff) << (8 * c);
    *reinterpret_cast<uint32_t*>(out + (int64_t)s * plane) = w;
  }
}

// v * 2^-e for the split (any finite v with |v| < 2^e): two exact multiplies
// by powers of two in the normal range
__device__ __forceinline__ double scale_down(double v, int e) {
  const int e1 = min(max(-e, -1022), 1023);
  const int e2 = min(max(-e - e1, -1022), 1023);
  return v * __hiloint2double((e1 + 1023) << 20, 0) * __hiloint2double((e2 + 1023) << 20, 0);
}

// One CTA per row of A: the row's largest magnitude gives ea (max < 2^ea),
// then each element is scaled into (-1, 1) and peeled.  Rows [m, mp) and
// columns [k, kp) are zeros; non-finite values raise the flag (they are
// split as zeros; the guarded fallback recomputes C).
template <class T>
__global__ void __launch_bounds__(256, 4)
ozaki_split_rows(int64_t m, int64_t k, int64_t kp, int64_t mp, const T* __restrict__ A,
                 int64_t lda, int S, int8_t* __restrict__ out, int* __restrict__ e_out,
                 int* __restrict__ flag, int digits8, int sign_gate) {
  __shared__ double red[8];
  const int64_t plane = mp * kp;
  for (int64_t i = blockIdx.x; i < mp; i += gridDim.x) {
    // sign gate: once any CTA saw a negative entry the split is moot
    if (sign_gate && *(volatile const int*)(flag + 1)) return;
    const T* arow = A + i * lda;
    double mx = 0.0;
    bool bad = false, neg = false;
    if (i < m) {
#pragma unroll 8
      for (int64_t j = threadIdx.x; j < k; j += blockDim.x) {   // 8 loads in flight per thread
        const double v = (double)arow[j];
        bad |= !isfinite(v);
        neg |= v < 0.0;
        mx = fmax(mx, fabs(v));
      }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(flag, 1);
    if (sign_gate && __syncthreads_or(neg)) {  // gate tripped: no digits needed
      if (threadIdx.x == 0) atomicExch(flag + 1, 1);
      return;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    mx = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, red[w]);
    __syncthreads();
    const int e = (mx > 0.0 && isfinite(mx)) ? ilogb(mx) + 1 : 0;
    if (threadIdx.x == 0 && i < m) e_out[i] = e;
    int8_t* orow = out + i * kp;
    // fp32 rows with a 16-byte pitch: one 16-byte load per 4 elements
    const bool vec4 = sizeof(T) == 4 && (lda % 4 == 0) && ((uintptr_t)A % 16 == 0);
#pragma unroll 2
    for (int64_t j = 4 * (int64_t)threadIdx.x; j < kp; j += 4 * (int64_t)blockDim.x) {
      double r[4];
      if (vec4 && i < m && j + 3 < k) {
        const float4 f = *reinterpret_cast<const float4*>(arow + j);
        const float fv[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) r[q] = isfinite(fv[q]) ? scale_down((double)fv[q], e) : 0.0;
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double v = (i < m && j + q < k) ? (double)arow[j + q] : 0.0;
          r[q] = isfinite(v) ? scale_down(v, e) : 0.0;
        }
      }
      if (digits8) peel4_u8(r[0], r[1], r[2], r[3], S, orow + j, plane);
      else if (S == 8 && (plane & 3) == 0) peel4_s8(r[0], r[1], r[2], r[3], orow + j, plane);
      else if (S <= 8 && (plane & 3) == 0) peel4_fast(r[0], r[1], r[2], r[3], S, orow + j, plane);
      else peel4(r[0], r[1], r[2], r[3], S, orow + j, plane);
    }
  }
}

// fp32 rows, 8-bit digits, S <= 3 (|floor(r 2^23)| < 2^23): the same digits
// as ozaki_split_rows in single-precision and 32-bit integer arithmetic — the
// scaling by 2^(7 + 8(S-1) - e) is two exact multiplies by powers of two (the
// product only rounds when it underflows, below the digits' resolution), one
// rounding-down conversion per element, byte planes by shifts; no fp64
// conversions and no 64-bit index arithmetic in the element loop
__device__ __forceinline__ float pow2f(int e) {   // 2^e for e in [-126, 127]
  return __int_as_float((e + 127) << 23);
}
__global__ void __launch_bounds__(256)
ozaki_split_rows_f32(int64_t m, int64_t k, int64_t kp, int64_t mp, const float* __restrict__ A,
                     int64_t lda, int S, int8_t* __restrict__ out, int* __restrict__ e_out,
                     int* __restrict__ flag, int sign_gate) {
  __shared__ float red[8];
  const int64_t plane = mp * kp;
  const int kk = (int)k, kpp = (int)kp;
  const bool vec4 = (lda % 4 == 0) && ((uintptr_t)A % 16 == 0) && (kk % 4 == 0);
  for (int64_t i = blockIdx.x; i < mp; i += gridDim.x) {
    if (sign_gate && *(volatile const int*)(flag + 1)) return;
    const float* arow = A + i * lda;
    float mx = 0.0f;
    bool bad = false, neg = false;
    if (i < m) {
      if (vec4) {
#pragma unroll 4
        for (int j = 4 * threadIdx.x; j < kk; j += 4 * blockDim.x) {
          const float4 f = *reinterpret_cast<const float4*>(arow + j);
          const float fv[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            bad |= !isfinite(fv[q]);
            neg |= fv[q] < 0.0f;
            mx = fmaxf(mx, fabsf(fv[q]));
          }
        }
      } else {
#pragma unroll 8
        for (int j = threadIdx.x; j < kk; j += blockDim.x) {
          const float v = arow[j];
          bad |= !isfinite(v);
          neg |= v < 0.0f;
          mx = fmaxf(mx, fabsf(v));
        }
      }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(flag, 1);
    if (sign_gate && __syncthreads_or(neg)) {
      if (threadIdx.x == 0) atomicExch(flag + 1, 1);
      return;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    mx = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = fmaxf(mx, red[w]);
    __syncthreads();
    const int e = (mx > 0.0f && isfinite(mx)) ? ilogbf(mx) + 1 : 0;
    if (threadIdx.x == 0 && i < m) e_out[i] = e;
    const int sh_all = 7 + 8 * (S - 1) - e;            // scale 2^sh_all = p1 * p2
    const int e1 = min(max(sh_all, -126), 127), e2 = min(max(sh_all - e1, -126), 127);
    const float p1 = pow2f(e1), p2 = pow2f(e2);
    uint32_t* o0 = reinterpret_cast<uint32_t*>(out + i * kp);
    for (int j = 4 * threadIdx.x; j < kpp; j += 4 * blockDim.x) {
      float fv[4];
      if (i < m && vec4 && j + 3 < kk) {
        const float4 f = *reinterpret_cast<const float4*>(arow + j);
        fv[0] = f.x; fv[1] = f.y; fv[2] = f.z; fv[3] = f.w;
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) fv[q] = (i < m && j + q < kk) ? arow[j + q] : 0.0f;
      }
      int qi[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) qi[q] = isfinite(fv[q]) ? __float2int_rd(fv[q] * p1 * p2) : 0;
      for (int s = 0; s < S; ++s) {
        const int sh = 8 * (S - 1 - s);
        uint32_t w = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) w |= (uint32_t)((qi[q] >> sh) & 0xff) << (8 * q);
        o0[(s * plane + j) >> 2] = w;
      }
    }
  }
}

// column magnitudes of B [k, n]: atomicMax on the bit pattern of |b| (monotone
// for non-negative doubles); NaN/inf raise the flag
template <class T>
__global__ void ozaki_colmax(int64_t k, int64_t n, const T* __restrict__ B, int64_t ldb,
                             unsigned long long* __restrict__ colmax, int* __restrict__ flag,
                             int sign_gate) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  if (sign_gate && *(volatile const int*)(flag + 1)) return;
  const int64_t k0 = (int64_t)blockIdx.y * 64, k1 = k0 + 64 < k ? k0 + 64 : k;
  double mx = 0.0;
  bool bad = false, neg = false;
  // 16 rows in flight per thread (8: 36.9 us for 4096^2 fp64, 87 % of the
  // warps' time on the load scoreboard; 16: 25.4 us)
#pragma unroll 16
  for (int64_t r = k0; r < k1; ++r) {
    const double v = (double)B[r * ldb + j];
    bad |= !isfinite(v);
    neg |= v < 0.0;
    mx = fmax(mx, fabs(v));
  }
  if (bad) atomicExch(flag, 1);
  if (sign_gate && neg) atomicExch(flag + 1, 1);
  atomicMax(colmax + j, (unsigned long long)__double_as_longlong(mx));
}

// B [k, n] -> digit planes [S][np][kp] (transposed: K-major).  A block stages
// 128 (k) x 32 (n) of B in shared memory; warp w then emits columns
// n0 + 4w .. 4w+3, lane l the 4 digits of k0 + 4l .. 4l+3: one 128-byte row
// segment per plane per warp store.
template <class T>
__global__ void __launch_bounds__(256)
ozaki_split_cols(int64_t k, int64_t n, int64_t kp, int64_t np, const T* __restrict__ B,
                 int64_t ldb, int S, const unsigned long long* __restrict__ colmax,
                 int8_t* __restrict__ out, int* __restrict__ e_out, int digits8,
                 const int* __restrict__ gate = nullptr) {
  if (gate && *(volatile const int*)gate) return;  // sign gate tripped (flag[1])
  // column c of row r lives at tile[r][c ^ (r / 4 % 32)]: the row-wise fill and
  // the 4-rows-per-lane column reads below are both free of bank conflicts
  __shared__ double tile[128][32];
  // a bounded grid walks the (n, k) tiles: a gated launch costs one wave
  const int64_t gxn = (np + 31) / 32, tiles = gxn * ((kp + 127) / 128);
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
  const int64_t by = t / gxn, bx = t % gxn;
  const int64_t k0 = by * 128, n0 = bx * 32;
  __syncthreads();   // the previous tile's reads of `tile` are done
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
#pragma unroll
  for (int r = ty; r < 128; r += 8) {
    const int64_t kk = k0 + r, nn = n0 + tx;
    const double v = (kk < k && nn < n) ? (double)B[kk * ldb + nn] : 0.0;
    tile[r][tx ^ ((r >> 2) & 31)] = isfinite(v) ? v : 0.0;
  }
  __syncthreads();
  const int64_t plane = np * kp;
  for (int c = 0; c < 4; ++c) {
    const int cc = 4 * ty + c;
    const int64_t nn = n0 + cc;
    const int64_t kk = k0 + 4 * tx;
    if (nn >= np || kk >= kp) continue;
    int e = 0;
    if (nn < n) {
      const double mx = __longlong_as_double((long long)colmax[nn]);
      e = (mx > 0.0 && isfinite(mx)) ? ilogb(mx) + 1 : 0;
      if (by == 0 && tx == 0) e_out[nn] = e;
    }
    double r[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) r[q] = (nn < n) ? scale_down(tile[4 * tx + q][cc ^ tx], e) : 0.0;
    if (digits8) peel4_u8(r[0], r[1], r[2], r[3], S, out + nn * kp + kk, plane);
    else if (S == 8 && (plane & 3) == 0) peel4_s8(r[0], r[1], r[2], r[3], out + nn * kp + kk, plane);
    else if (S <= 8 && (plane & 3) == 0) peel4_fast(r[0], r[1], r[2], r[3], S, out + nn * kp + kk, plane);
    else peel4(r[0], r[1], r[2], r[3], S, out + nn * kp + kk, plane);
  }
  }
}

// fp32 B, 8-bit digits, S <= 3: ozaki_colmax / ozaki_split_cols in single
// precision (see ozaki_split_rows_f32); the column maxima are kept as the
// fp64 bit patterns the fp64 kernels use
__global__ void ozaki_colmax_f32(int64_t k, int64_t n, const float* __restrict__ B, int64_t ldb,
                                 unsigned long long* __restrict__ colmax, int* __restrict__ flag,
                                 int sign_gate) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  if (sign_gate && *(volatile const int*)(flag + 1)) return;
  const int64_t k0 = (int64_t)blockIdx.y * 64, k1 = k0 + 64 < k ? k0 + 64 : k;
  float mx = 0.0f;
  bool bad = false, neg = false;
  const float* col = B + j;
#pragma unroll 16
  for (int64_t r = k0; r < k1; ++r) {
    const float v = col[r * ldb];
    bad |= !isfinite(v);
    neg |= v < 0.0f;
    mx = fmaxf(mx, fabsf(v));
  }
  if (bad) atomicExch(flag, 1);
  if (sign_gate && neg) atomicExch(flag + 1, 1);
  atomicMax(colmax + j, (unsigned long long)__double_as_longlong((double)mx));
}

__global__ void __launch_bounds__(256)
ozaki_split_cols_f32(int64_t k, int64_t n, int64_t kp, int64_t np, const float* __restrict__ B,
                     int64_t ldb, int S, const unsigned long long* __restrict__ colmax,
                     int8_t* __restrict__ out, int* __restrict__ e_out,
                     const int* __restrict__ gate = nullptr) {
  if (gate && *(volatile const int*)gate) return;
  __shared__ float tile[128][32];   // column c of row r at [r][c ^ (r / 4 % 32)]: conflict-free
  __shared__ float sc1[32], sc2[32];  // per-column scale factors 2^e1, 2^e2
  const int64_t gxn = (np + 31) / 32, tiles = gxn * ((kp + 127) / 128);
  const int64_t plane4 = np * kp / 4;   // digit plane stride in 32-bit words
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
  const int ldb32 = (int)ldb;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int64_t by = t / gxn, bx = t % gxn;
    const int64_t k0 = by * 128, n0 = bx * 32;
    const int krem = (int)min((int64_t)128, k - k0), nrem = (int)min((int64_t)32, n - n0);
    __syncthreads();
    if (ty == 0) {   // the column's exponent (from the maxima of ozaki_colmax_f32) and scales
      int e = 0;
      if (tx < nrem) {
        const double mx = __longlong_as_double((long long)colmax[n0 + tx]);
        e = (mx > 0.0 && isfinite(mx)) ? ilogb(mx) + 1 : 0;
        if (by == 0) e_out[n0 + tx] = e;
      }
      const int sh_all = 7 + 8 * (S - 1) - e;
      const int e1 = min(max(sh_all, -126), 127), e2 = min(max(sh_all - e1, -126), 127);
      sc1[tx] = pow2f(e1);
      sc2[tx] = pow2f(e2);
    }
    const float* __restrict__ tb = B + k0 * ldb + n0;   // 32-bit offsets inside the tile
#pragma unroll 8
    for (int r = ty; r < 128; r += 8) {
      const float v = (r < krem && tx < nrem) ? tb[r * ldb32 + tx] : 0.0f;
      tile[r][tx ^ ((r >> 2) & 31)] = isfinite(v) ? v : 0.0f;
    }
    __syncthreads();
    const bool kin = k0 + 4 * tx < kp;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int cc = 4 * ty + c;
      if (n0 + cc >= np || !kin) continue;
      const float p1 = sc1[cc], p2 = sc2[cc];
      const bool live = cc < nrem;
      int qi[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        qi[q] = live ? __float2int_rd(tile[4 * tx + q][cc ^ tx] * p1 * p2) : 0;
      uint32_t* o = reinterpret_cast<uint32_t*>(out + (n0 + cc) * kp + k0) + tx;
      for (int s2 = 0; s2 < S; ++s2) {
        const int sh = 8 * (S - 1 - s2);
        uint32_t w = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) w |= (uint32_t)((qi[q] >> sh) & 0xff) << (8 * q);
        o[s2 * plane4] = w;
      }
    }
  }
}

// sign gate probe: any negative among the first `rows` rows of A and of B
// raises flag[1] before the split kernels start (mixed-sign operands then
// skip the digit split at the cost of one small read)
template <class T>
__global__ void ozaki_sign_probe(int64_t m, int64_t k, const T* __restrict__ A, int64_t lda,
                                 int64_t kb, int64_t n, const T* __restrict__ B, int64_t ldb,
                                 int64_t rows, int* __restrict__ flag) {
  // CTA c < rows: row c of A; rows <= c < 2 rows: row c - rows of B
  bool neg = false;
  const int64_t c = blockIdx.x;
  if (c < rows && c < m) {
    for (int64_t j = threadIdx.x; j < k; j += blockDim.x) neg |= A[c * lda + j] < T(0);
  } else if (c >= rows && c - rows < kb) {
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) neg |= B[(c - rows) * ldb + j] < T(0);
  }
  if (__syncthreads_or(neg) && threadIdx.x == 0) atomicExch(flag + 1, 1);
}

// -------------------------------------------------------------- host side
static int make_i8_map(CUtensorMap* map, const int8_t* base, int64_t rows, int64_t kp,
                       uint32_t box_rows) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(LAPIS_B200_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {(cuuint64_t)kp, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)kp};
  const cuuint32_t box[2] = {(cuuint32_t)OZ_BK, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(LAPIS_B200_ERR_CUDA, "cuTensorMapEncodeTiled (int8) failed");
  return LAPIS_B200_OK;
}

// S digit planes [S][rows][kp] as one 3-D map: box {32, box_rows, box_digits}, SWIZZLE_32B
static int make_i8_map3(CUtensorMap* map, const int8_t* base, int64_t rows, int64_t kp, int S,
                        uint32_t box_rows, uint32_t box_digits) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(LAPIS_B200_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[3] = {(cuuint64_t)kp, (cuuint64_t)rows, (cuuint64_t)S};
  const cuuint64_t strides[2] = {(cuuint64_t)kp, (cuuint64_t)(rows * kp)};
  const cuuint32_t box[3] = {32u, box_rows, box_digits};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(LAPIS_B200_ERR_CUDA, "cuTensorMapEncodeTiled (int8, 3-D) failed");
  return LAPIS_B200_OK;
}

// Digits per operand for a k-deep product, 0 when the scheme cannot certify
// the contract for unit-scale data (or s32 accumulation would overflow):
// fp64 7-bit digits, per-product bound (S + 1) 2^-7S -> S = 8 up to k ~ 6000,
// S = 9 up to the s32 limit; fp32 8-bit digits, S = 3 up to the s32 limit.
int ozaki_slices_for(int dtype, int64_t k) {
  if (dtype == LAPIS_B200_F64) {
    if (k * 9.0 * ldexp(1.0, -56) <= 0.75e-12 && 8 * k * 16129 < (1ll << 31)) return 8;
    if (k * 10.0 * ldexp(1.0, -63) <= 0.75e-12 && 9 * k * 16129 < (1ll << 31)) return 9;
    return 0;
  }
  if (dtype == LAPIS_B200_F32 && 3 * k * 65025 < (1ll << 31)) return 3;
  return 0;
}

template <class T>
static int launch_ozaki_2p(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mb64,
                           const OzParams& prm, int grid, cudaStream_t st) {
  // fp64: two passes, 8 digits; fp32: one pass, 3 digits of 8 bits.  Clusters
  // share operand boxes: pairs along m by default; LAPIS_B200_OZAKI_CLUSTER =
  // 0 (single CTAs) or 4 (2 x 2, A and B shared: only 34 of 37 clusters are
  // co-resident, 4096^3 f64 1.99 vs 1.88 ms with pairs, f32 0.511 vs 0.508)
  static const int cl_env = [] {
    const char* e = getenv("LAPIS_B200_OZAKI_CLUSTER");
    return e ? atoi(e) : 2;
  }();
  int cmn = 1;
  if (cl_env >= 4 && prm.num_m % 2 == 0 && prm.num_n % 2 == 0) cmn = 4;
  else if (cl_env >= 2 && prm.num_m % 2 == 0) cmn = 2;
  constexpr bool F64 = std::is_same<T, double>::value;
  // the m-pairs run cta_group::2 MMAs (M = 256): fp64 4096^3 1.89 -> 1.79
  // ms; fp32 (after the integer epilogue combine) 0.4754 -> 0.4730 ms;
  // LAPIS_B200_OZAKI_PAIR = 0 keeps per-CTA MMAs in the clusters
  static const int pair_env = [] {
    const char* e = getenv("LAPIS_B200_OZAKI_PAIR");
    return e ? atoi(e) : 1;
  }();
  const bool pair = cmn == 2 && pair_env == 1;
  auto kern = pair ? (F64 ? gemm_ozaki_2p_kernel<double, 2, 8, false, 2, 1, true>
                          : gemm_ozaki_2p_kernel<float, 1, 3, true, 2, 1, true>)
            : cmn == 4 ? (F64 ? gemm_ozaki_2p_kernel<double, 2, 8, false, 2, 2>
                              : gemm_ozaki_2p_kernel<float, 1, 3, true, 2, 2>)
            : cmn == 2 ? (F64 ? gemm_ozaki_2p_kernel<double, 2, 8, false, 2, 1>
                              : gemm_ozaki_2p_kernel<float, 1, 3, true, 2, 1>)
                       : (F64 ? gemm_ozaki_2p_kernel<double, 2, 8, false, 1, 1>
                              : gemm_ozaki_2p_kernel<float, 1, 3, true, 1, 1>);
  LB_TRY(check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)OZ2_SMEM), "smem attr (gemm_ozaki_2p_kernel)"));
  if (cmn == 1) {
    kern<<<grid, OZ_THREADS, OZ2_SMEM, st>>>(ma, mb, prm);
    return check_launch("gemm_ozaki_2p_kernel");
  }
  const int units = (prm.num_m / (cmn == 4 ? 2 : 2)) * (prm.num_n / (cmn == 4 ? 2 : 1));
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(OZ_THREADS, 1, 1);
  cfg.dynamicSmemBytes = OZ2_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)cmn;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // one resident wave of clusters: clusters must fit inside a GPC, so fewer
  // than #SMs / cmn may be co-resident
  int max_clusters = grid / cmn;
  cfg.gridDim = dim3((unsigned)(cmn * max_clusters), 1, 1);
  int active = 0;
  if (cudaOccupancyMaxActiveClusters(&active, (void*)kern, &cfg) == cudaSuccess && active > 0)
    max_clusters = std::min(max_clusters, active);
  cudaGetLastError();
  int gc = std::min(units, max_clusters);
  if (gc < 1) gc = 1;
  cfg.gridDim = dim3((unsigned)(cmn * gc), 1, 1);
  LB_TRY(check_cuda(cudaLaunchKernelEx(&cfg, kern, ma, pair ? mb64 : mb, prm),
                    "launch (gemm_ozaki_2p_kernel, cluster)"));
  return check_launch("gemm_ozaki_2p_kernel");
}

// TWO_PASS: the two-pass kernel (fp64, S = 8, BN = 128)
template <class T, int BN, bool TWO_PASS = false>
static int gemm_ozaki_t(int64_t batch, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda,
                        const void* B, int64_t ldb, void* C, int64_t ldc, int64_t sA, int64_t sB,
                        int64_t sC, int S, cudaStream_t st, int sign_gate = 0) {
  if (m > 0x7fffffff || n > 0x7fffffff || k > 0x7fffffff)
    return fail(LAPIS_B200_ERR_ARG, "gemm ozaki: extent too large");
  if (S < 1 || S > OZ_MAX_S) return fail(LAPIS_B200_ERR_ARG, "gemm ozaki: bad slice count");
  // fp32: 8-bit digits (signed leading + unsigned), S = 3 covers 24 bits;
  // fp64: 7-bit signed digits (truncation toward zero keeps the dropped
  // remainders sign-symmetric, which the 1e-12 contract needs), S = 8
  const int digits8 = std::is_same<T, float>::value ? 1 : 0;
  const int64_t dmax = digits8 ? 255 * 255 : 127 * 127;
  // int32 accumulation bound: (d+1) * k * max|digit product| < 2^31 for every diagonal
  if ((int64_t)S * k * dmax >= (1ll << 31))
    return fail(LAPIS_B200_ERR_UNSUPPORTED, "gemm ozaki: k too large for s32 accumulation");
  constexpr int64_t DT = std::is_same<T, double>::value ? LAPIS_B200_F64 : LAPIS_B200_F32;
  const int dtype = (int)DT;
  if (k == 0) return launch_gemm_exact_guarded(m, n, k, A, lda, B, ldb, C, ldc, dtype, Guard(), st);
  static thread_local int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if constexpr (!TWO_PASS) {
    if (configured_dev != dev) {
      LB_TRY(check_cuda(cudaFuncSetAttribute(gemm_ozaki_kernel<T, BN>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)OzTile<BN>::SMEM),
                        "smem attr (gemm_ozaki_kernel)"));
      configured_dev = dev;
    }
  }
  const int64_t kp = (k + 15) / 16 * 16;
  const int64_t mp = (m + OZ_BM - 1) / OZ_BM * OZ_BM, np = (n + BN - 1) / BN * BN;
  // workspace: digits of A and B, exponents, column maxima, flag, fp32 partials
  const size_t a_bytes = (size_t)S * mp * kp, b_bytes = (size_t)S * np * kp;
  const size_t part_bytes = (std::is_same<T, float>::value && !TWO_PASS) ? (size_t)m * n * sizeof(double) : 0;
  const size_t meta = (size_t)(m + n) * sizeof(int) + (size_t)n * 8 + 64 + 8;
  // last-wave split: with R tiles left after the full waves and 2R <= #SMs,
  // each of them is cut in two halves of about equal int8 work
  const int num_m_t = (int)(mp / OZ_BM), num_n_t = (int)(np / BN);
  const int tiles = num_m_t * num_n_t, sms = num_sms();
  static const bool split_on = [] {
    const char* e = getenv("LAPIS_B200_OZAKI_SPLIT");
    return !(e && e[0] == '0');
  }();
  const int rem = tiles % sms;
  const int nsplit = (!TWO_PASS && split_on && S > 1 && rem > 0 && 2 * rem <= sms) ? rem : 0;
  const int grid = nsplit ? (tiles >= sms ? sms : 2 * rem) : std::min(tiles, sms);
  uint32_t helper_mask = 0;
  if (nsplit) {
    // helper: the subset of diagonals 0..S-2 (diagonal d = d+1 slice products)
    // minimising the larger half
    const int all = S * (S + 1) / 2;
    int best = all;
    for (uint32_t msk = 1; msk < (1u << (S - 1)); ++msk) {
      int h = 0;
      for (int d = 0; d < S - 1; ++d) h += ((msk >> d) & 1u) ? d + 1 : 0;
      const int mx = std::max(h, all - h);
      if (mx < best) { best = mx; helper_mask = msk; }
    }
  }
  const size_t split_bytes = TWO_PASS ? (size_t)std::min(tiles, sms) * OZ2_SLOT * sizeof(double)
                          : nsplit ? (size_t)nsplit * OZ_BM * BN * sizeof(double) : 0;
  const size_t flag_bytes = (size_t)nsplit * OZ_EPI_WARPS * sizeof(int);
  uint8_t* ws = nullptr;
  LB_TRY(check_cuda(cudaMallocAsync((void**)&ws, a_bytes + b_bytes + part_bytes + split_bytes +
                                                     meta + flag_bytes + 512, st),
                    "alloc(ozaki workspace)"));
  int8_t* ad = reinterpret_cast<int8_t*>(ws);
  int8_t* bd = ad + a_bytes;
  double* part = reinterpret_cast<double*>(ws + ((a_bytes + b_bytes + 255) / 256 * 256));
  double* split_ws = reinterpret_cast<double*>(
      (reinterpret_cast<uintptr_t>(part) + part_bytes + 255) / 256 * 256);
  uint8_t* mp_ = reinterpret_cast<uint8_t*>(split_ws) + split_bytes;
  unsigned long long* colmax = reinterpret_cast<unsigned long long*>(mp_);
  int* ea = reinterpret_cast<int*>(colmax + n);
  int* eb = ea + m;
  int* flag = eb + n;
  int* split_flag = flag + 2;
  int rc = LAPIS_B200_OK;
  for (int64_t b = 0; b < batch && rc == LAPIS_B200_OK; ++b) {
    const T* Ab = (const T*)A + b * sA;
    const T* Bb = (const T*)B + b * sB;
    T* Cb = (T*)C + b * sC;
    // column maxima, exponents and flags are contiguous: one memset
    rc = check_cuda(cudaMemsetAsync(colmax, 0,
                                    (size_t)(reinterpret_cast<uint8_t*>(flag) -
                                             reinterpret_cast<uint8_t*>(colmax)) +
                                        2 * sizeof(int) + flag_bytes, st),
                    "memset(colmax, flags)");
    if (rc != LAPIS_B200_OK) break;
    const int64_t rblocks = std::min<int64_t>(mp, (int64_t)num_sms() * 16);
    if (sign_gate)
      ozaki_sign_probe<T><<<2 * 64, 256, 0, st>>>(m, k, Ab, lda, k, n, Bb, ldb, 64, flag);
    // A's row split and B's column passes are independent: B's run on a
    // forked stream (joined before the product kernel), so the two
    // issue/latency-bound passes share the machine (LAPIS_B200_OZAKI_FORK=0:
    // one stream)
    cudaStream_t sb = st;
    static const bool fork_on = [] {
      const char* e = getenv("LAPIS_B200_OZAKI_FORK");
      return !(e && e[0] == '0');
    }();
    static thread_local cudaStream_t side[64] = {};
    static thread_local cudaEvent_t ev_fork[64] = {}, ev_join[64] = {};
    int sdev = 0;
    cudaGetDevice(&sdev);
    if (fork_on && sdev >= 0 && sdev < 64) {
      if (!side[sdev] &&
          (cudaStreamCreateWithFlags(&side[sdev], cudaStreamNonBlocking) != cudaSuccess ||
           cudaEventCreateWithFlags(&ev_fork[sdev], cudaEventDisableTiming) != cudaSuccess ||
           cudaEventCreateWithFlags(&ev_join[sdev], cudaEventDisableTiming) != cudaSuccess))
        side[sdev] = nullptr;
      if (side[sdev] && cudaEventRecord(ev_fork[sdev], st) == cudaSuccess &&
          cudaStreamWaitEvent(side[sdev], ev_fork[sdev], 0) == cudaSuccess)
        sb = side[sdev];
      cudaGetLastError();
    }
    if constexpr (std::is_same<T, float>::value) {
      if (digits8 && S <= 3 && kp % 4 == 0 && (mp * kp) % 4 == 0)
        ozaki_split_rows_f32<<<(unsigned)rblocks, 256, 0, st>>>(m, k, kp, mp, Ab, lda, S, ad, ea, flag,
                                                                sign_gate);
      else
        ozaki_split_rows<T><<<(unsigned)rblocks, 256, 0, st>>>(m, k, kp, mp, Ab, lda, S, ad, ea, flag,
                                                               digits8, sign_gate);
    } else {
      ozaki_split_rows<T><<<(unsigned)rblocks, 256, 0, st>>>(m, k, kp, mp, Ab, lda, S, ad, ea, flag,
                                                             digits8, sign_gate);
    }
    dim3 cg((unsigned)((n + 255) / 256), (unsigned)((k + 63) / 64));
    const int64_t tg = ((np + 31) / 32) * ((kp + 127) / 128);
    bool f32fast = false;
    if constexpr (std::is_same<T, float>::value) f32fast = digits8 && S <= 3;
    if (f32fast) {
      ozaki_colmax_f32<<<cg, 256, 0, sb>>>(k, n, (const float*)Bb, ldb, colmax, flag, sign_gate);
      ozaki_split_cols_f32<<<(unsigned)tg, 256, 0, sb>>>(k, n, kp, np, (const float*)Bb, ldb, S, colmax,
                                                         bd, eb, sign_gate ? flag + 1 : nullptr);
    } else {
      ozaki_colmax<T><<<cg, 256, 0, sb>>>(k, n, Bb, ldb, colmax, flag, sign_gate);
      ozaki_split_cols<T><<<(unsigned)tg, 256, 0, sb>>>(k, n, kp, np, Bb, ldb, S, colmax, bd, eb,
                                                        digits8, sign_gate ? flag + 1 : nullptr);
    }
    rc = check_launch("ozaki split");
    if (sb != st) {
      const int jrc = check_cuda(cudaEventRecord(ev_join[sdev], sb), "record(ozaki join)");
      const int wrc = check_cuda(cudaStreamWaitEvent(st, ev_join[sdev], 0), "wait(ozaki join)");
      if (rc == LAPIS_B200_OK) rc = jrc != LAPIS_B200_OK ? jrc : wrc;
    }
    CUtensorMap ma, mb;
    if (TWO_PASS) {
      if (rc == LAPIS_B200_OK) rc = make_i8_map3(&ma, ad, mp, kp, S, OZ_BM, S < 4 ? S : 4);
      if (rc == LAPIS_B200_OK) rc = make_i8_map3(&mb, bd, np, kp, S, BN, S < 4 ? S : 4);
    } else {
      if (rc == LAPIS_B200_OK) rc = make_i8_map(&ma, ad, (int64_t)S * mp, kp, OZ_BM);
      if (rc == LAPIS_B200_OK) rc = make_i8_map(&mb, bd, (int64_t)S * np, kp, BN);
    }
    if (rc != LAPIS_B200_OK) break;
    OzParams prm;
    prm.m = (int)m;
    prm.n = (int)n;
    prm.nk = (int)((kp + OZ_BK - 1) / OZ_BK);
    prm.num_m = num_m_t;
    prm.num_n = num_n_t;
    prm.split_base = nsplit ? (tiles / sms) * grid : tiles;
    prm.nsplit = nsplit;
    prm.helper_mask = helper_mask;
    prm.owner_mask = ((1u << S) - 1u) & ~helper_mask;
    prm.split_ws = split_ws;
    prm.split_flag = split_flag;
    prm.S = S;
    prm.mp = (int)mp;
    prm.np = (int)np;
    prm.C = Cb;
    prm.ldc = ldc;
    prm.part = std::is_same<T, double>::value ? reinterpret_cast<double*>(Cb) : part;
    prm.ldp = std::is_same<T, double>::value ? ldc : n;
    prm.ea = ea;
    prm.eb = eb;
    prm.flag = flag;
    {
      // a-priori bound per product, in units of 2^(ea_i + eb_j): the digit
      // truncation of both operands (2 delta) plus the dropped digit products
      // (s + t >= S); K products; 3/4 of the contract certified, the rest left
      // for the reference's own rounding
      const double delta = digits8 ? ldexp(1.0, -(7 + 8 * (S - 1))) : ldexp(1.0, -7 * S);
      const double cross = digits8 ? (S - 1) * ldexp(1.0, 2 - 8 * S) : (S - 1) * ldexp(1.0, -7 * S);
      prm.cert_k = (double)k * (2.0 * delta + delta * delta + cross) * (1.0 + 1e-3);
      prm.cert_tol = 0.75 * (std::is_same<T, double>::value ? 1e-12 : 1e-5);
    }
    prm.digits8 = digits8;
    prm.sign_gate = sign_gate;
    prm.vec2 = (prm.ldp % 2 == 0) && ((uintptr_t)prm.part % 16 == 0);
    static const bool prof_on = [] {
      const char* e = getenv("LAPIS_B200_OZAKI_PROF");
      return e && e[0] == '1';
    }();
    unsigned long long* dprof = nullptr;
    if (prof_on) {
      cudaMallocAsync((void**)&dprof, 8 * sizeof(unsigned long long), st);
      cudaMemsetAsync(dprof, 0, 8 * sizeof(unsigned long long), st);
    }
    prm.prof = dprof;
    if constexpr (TWO_PASS) {
      prm.nk = (int)((kp + OZ2_BK - 1) / OZ2_BK);
      prm.vec2 = ((uintptr_t)Cb % (2 * sizeof(T)) == 0) && (ldc % 2 == 0);
      CUtensorMap mb64;   // B boxes of 64 rows: each CTA of a cta_group::2 pair stages half the tile
      rc = make_i8_map3(&mb64, bd, np, kp, S, 64, S < 4 ? S : 4);
      if (rc == LAPIS_B200_OK) rc = launch_ozaki_2p<T>(ma, mb, mb64, prm, std::min(tiles, sms), st);
    } else {
      gemm_ozaki_kernel<T, BN><<<grid, OZ_THREADS, OzTile<BN>::SMEM, st>>>(ma, mb, prm);
      rc = check_launch("gemm_ozaki_kernel");
    }
    if (dprof) {
      unsigned long long h[8];
      cudaMemcpyAsync(h, dprof, sizeof(h), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      fprintf(stderr, "ozaki prof (cycles summed over CTAs): producer-wait-empty %llu  "
              "mma-wait-tmem-empty %llu  mma-wait-full %llu  mma-total %llu  epi-wait-full %llu  "
              "drain %llu over %llu drains (%.0f cycles each)\n",
              h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[6] ? (double)h[5] / h[6] : 0.0);
      cudaFreeAsync(dprof, st);
    }
    // non-finite inputs: the reference-order GEMM, run only when flag[0] is set;
    // a certification failure (flag[1]): the fp64 DMMA / fp32 3xTF32 path
    if (rc == LAPIS_B200_OK)
      rc = launch_gemm_exact_guarded(m, n, k, Ab, lda, Bb, ldb, Cb, ldc, dtype, Guard{flag, 1}, st);
    if (rc == LAPIS_B200_OK) {
      if (std::is_same<T, double>::value)
        rc = gemm_dmma(1, m, n, k, Ab, lda, Bb, ldb, Cb, ldc, 0, 0, 0, st, Guard{flag, 2});
      else
        rc = gemm_tf32x3(1, m, n, k, Ab, lda, Bb, ldb, Cb, ldc, 0, 0, 0, st, Guard{flag, 2});
    }
  }
  cudaFreeAsync(ws, st);
  return rc;
}

int gemm_ozaki(int64_t batch, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda,
               const void* B, int64_t ldb, void* C, int64_t ldc, int64_t sA, int64_t sB,
               int64_t sC, int dtype, int slices, cudaStream_t st, int sign_gate) {
  const int S = slices > 0 ? slices : ozaki_slices_for(dtype, k);
  if (S == 0) return fail(LAPIS_B200_ERR_UNSUPPORTED, "gemm ozaki: k out of the certified range");
  static const int bn_env = [] {
    const char* e = getenv("LAPIS_B200_OZAKI_BN");
    return e ? atoi(e) : 0;
  }();
  const int bn = bn_env ? bn_env : (dtype == LAPIS_B200_F64 ? 256 : 192);
  // fp64 S = 8: the two-pass kernel (LAPIS_B200_OZAKI_2P=0 selects the
  // per-diagonal kernel)
  static const bool two_pass = [] {
    const char* e = getenv("LAPIS_B200_OZAKI_2P");
    return !(e && e[0] == '0');
  }();
  if (two_pass && dtype == LAPIS_B200_F64 && S == 8)
    return gemm_ozaki_t<double, OZ2_BN, true>(batch, m, n, k, A, lda, B, ldb, C, ldc, sA, sB, sC, S, st);
  // fp32, S = 3 through the same kernel in one pass (LAPIS_B200_OZAKI_1P=1):
  // correct, but 0.747 vs 0.595 ms for the per-diagonal kernel at 4096^3 — the
  // three diagonals fill 384 TMEM columns, so each tile's drain stalls the
  // MMAs, while the per-diagonal kernel double-buffers its accumulators
  static const bool one_pass = [] {
    const char* e = getenv("LAPIS_B200_OZAKI_1P");
    return !(e && e[0] == '0');
  }();
  if (one_pass && dtype == LAPIS_B200_F32 && S == 3)
    return gemm_ozaki_t<float, OZ2_BN, true>(batch, m, n, k, A, lda, B, ldb, C, ldc, sA, sB, sC, S, st,
                                             sign_gate);
#define LB_OZ(T, BN_) return gemm_ozaki_t<T, BN_>(batch, m, n, k, A, lda, B, ldb, C, ldc, sA, sB, sC, S, st, sign_gate)
  if (dtype == LAPIS_B200_F64) { if (bn == 192) LB_OZ(double, 192); LB_OZ(double, 256); }
  if (dtype == LAPIS_B200_F32) { if (bn == 256) LB_OZ(float, 256); LB_OZ(float, 192); }
#undef LB_OZ
  return fail(LAPIS_B200_ERR_UNSUPPORTED, "gemm ozaki: f32 / f64 only");
}

}  // namespace lapis_b200
