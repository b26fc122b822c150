/*
 * lapis_b200.h — C ABI of the B200 (sm_100a) execution backend for the LAPIS
 * hot path: CSR SpMV, CSR x dense SpMM, dense matmul / matvec /
 * batch_matmul, and the parallel_reduce family.
 *
 * The reference (arXiv 2509.25605, /root/reference) executes these kernels as
 * emitted Kokkos C++ on a serial stub; its "FFI" is the emitted C++ signature
 * plus the runtime-header library seam.  Each entry below replaces one of
 * those, cited as reference file:line.  Conventions:
 *
 *   - all buffer pointers are DEVICE pointers (the "unmanaged View" analogue)
 *     in row-major LayoutRight (runtime_header.py:39-41); the caller owns them
 *     and the library keeps none of them after return (plans excepted);
 *   - outputs (y, Y, C) are overwritten, never accumulated (interp.py:812);
 *   - `stream` is a cudaStream_t (NULL = legacy default stream); every call is
 *     stream-ordered and asynchronous, nothing synchronises the device;
 *   - return 0 on success, a LAPIS_B200_ERR_* code otherwise, with a
 *     thread-local message in lapis_b200_last_error(); the host process is
 *     never aborted (the reference stub calls exit(1),
 *     lapis_serial_stub.hpp:29-32);
 *   - threads: any number of host threads may call concurrently, each on its
 *     own stream (per-call scratch comes from stream-ordered cudaMallocAsync;
 *     plans are read-only after creation); tests/test_threads_gpu.py;
 *   - scratch memory: the first call on a device raises the release threshold
 *     of that device's DEFAULT memory pool so per-call workspaces stay cached
 *     in the pool (a process-wide setting other cudaMallocAsync users share);
 *     LAPIS_B200_KEEP_POOL=0 leaves the pool as the caller configured it.
 */
#ifndef LAPIS_B200_H
#define LAPIS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define LAPIS_B200_OK 0
#define LAPIS_B200_ERR_ARG 1         /* bad argument (shape, pointer, dtype) */
#define LAPIS_B200_ERR_CUDA 2        /* CUDA runtime / launch error */
#define LAPIS_B200_ERR_UNSUPPORTED 3 /* dtype / mode combination not provided */
#define LAPIS_B200_ERR_NOMEM 4       /* device allocation failed */

/* element types: the reference's scalar kinds f32, f64, i32, i64/index
 * (ir.py:23-92; index is 64-bit, emitter.py:39-42) */
#define LAPIS_B200_F32 0
#define LAPIS_B200_F64 1
#define LAPIS_B200_I32 2
#define LAPIS_B200_I64 3

/* reduction combiners (dialect.py:128-154 classify_combiner; identities
 * interp.py:186-195) */
#define LAPIS_B200_ADD 0
#define LAPIS_B200_MUL 1
#define LAPIS_B200_MIN 2
#define LAPIS_B200_MAX 3

/* dense matmul precision modes (lapis_b200_gemm `mode`) */
#define LAPIS_B200_GEMM_AUTO 0    /* f32 -> OZAKI when A and B hold no negative entry
                                     (checked on the device; any negative entry, or a
                                     failed certificate, recomputes with TF32X3) and k is in
                                     its range, TF32X3 otherwise; f64 -> OZAKI (DMMA beyond
                                     its k range); ints -> EXACT */
#define LAPIS_B200_GEMM_TF32X3 1  /* f32: 3xTF32 split on tcgen05 (kind::tf32), TMEM accum */
#define LAPIS_B200_GEMM_DMMA 2    /* f64: DMMA tensor cores */
#define LAPIS_B200_GEMM_EXACT 3   /* reference order: sequential k, no FMA -> bit-exact */
#define LAPIS_B200_GEMM_OZAKI 4   /* f64 / f32: Ozaki digit split on the int8 tensor cores
                                     (tcgen05 kind::i8; f64 8-9 7-bit digits, f32 3 8-bit
                                     digits; s32 accumulation).  Every element is certified
                                     against an a-priori error bound; uncertified results
                                     are recomputed by DMMA / TF32X3 on the device */

/* ----------------------------------------------------------------- library */
const char* lapis_b200_last_error(void);
int lapis_b200_version(void);
/* Diagnostics (not a reference interface): the kernel nodes of a captured
 * cudaGraph_t, one mangled name per line into buf (NUL-terminated, truncated
 * to cap), their count in *nkernels — the bench's launch census of a step. */
int lapis_b200_graph_kernels(void* graph, char* buf, int64_t cap, int64_t* nkernels);
/* Select and warm up `device` for the calling thread (lapis_initialize,
 * golden/cpp/spmv.hpp:8-10). */
int lapis_b200_init(int device);
/* Release cached per-device workspaces (lapis_finalize, spmv.hpp:12-14). */
int lapis_b200_finalize(void);

/* The CSR vector-length hint the reference computes before every SpMV:
 * min(nextPow2(ceil(nnz / max(nrows, 1))), max_vector_length)
 * (loop_mapping.py:224-246; emitted as golden/cpp/spmv.hpp:17-33).  Host-only. */
int64_t lapis_b200_csr_vector_length(int64_t nrows, int64_t nnz, int64_t max_vector_length);

/* ------------------------------------------------------------- sparse.spmv_csr
 * y[i] = sum_{j in [rowptr[i], rowptr[i+1])} values[j] * x[colind[j]]
 * Replaces the emitted `spmv(rowptr, colind, values, x, y)`
 * (tests/golden/cpp/spmv.hpp:16-70, op contract dialect.py:222,797-812,
 * semantics interp.py:798-812).
 *   rowptr_bytes, colind_bytes in {4, 8} (i32 or i64/index);
 *   dtype in {F32, F64, I32, I64} for values / x / y;
 *   vector_length = 0: a device-side choice, no host round trip: one pass over
 *     rowptr (longest row, monotonicity), then regular structures run the
 *     vector-lane kernel in exact mode (every row bit-identical), irregular
 *     ones the warp-block kernel and non-monotone rowptrs the tiled row-stream
 *     kernel (both: rows up to 512 entries summed in ascending order,
 *     bit-identical; longer fp64 rows as a fixed tree, within tolerance);
 *   vector_length = 1..32 (power of two): the emitted TeamPolicy mapping with
 *     that vector length (one row per `vector_length` lanes, shuffle tree). */
int lapis_b200_spmv_csr(int64_t nrows, int64_t ncols, int64_t nnz,
                        const void* rowptr, int rowptr_bytes,
                        const void* colind, int colind_bytes,
                        const void* values, const void* x, void* y,
                        int dtype, int vector_length, void* stream);

/* A CSR "plan": structure-only analysis (tile -> first-row table of the tiled
 * kernel) cached across calls on the same rowptr, the analogue of hoisting
 * the rowptr-derived vector length out of the call.  The plan
 * keeps a device allocation until lapis_b200_csr_plan_destroy. */
typedef struct lapis_b200_csr_plan_s* lapis_b200_csr_plan;
int lapis_b200_csr_plan_create(int64_t nrows, int64_t nnz, const void* rowptr, int rowptr_bytes,
                               void* stream, lapis_b200_csr_plan* out_plan);
int lapis_b200_csr_plan_destroy(lapis_b200_csr_plan plan);
int lapis_b200_spmv_csr_plan(lapis_b200_csr_plan plan, const void* rowptr, int rowptr_bytes,
                             const void* colind, int colind_bytes, const void* values,
                             const void* x, void* y, int dtype, void* stream);
/* What the analysis chose: out[0] = longest row, out[1] = vector length of the
 * vector-lane kernel (0 = row-stream tile kernel), out[2] = number of tiles,
 * out[3] = flags: bit 0 exact mode, bit 1 warp-block kernel, bit 2 the
 * row-stream kernel (regular rows of 15-28 entries: each tile's row offsets,
 * colind and values staged by TMA bulk copies, one row per thread, tiles
 * handed out in runs of 5 by a device counter), bit 3 the row-stream kernel in
 * every mode (its sequential row sums are the reference's bits; default for
 * such structures, LAPIS_B200_RS_TREE=0 keeps the vector kernel in tree
 * mode).  Other regular structures (longest row <= max(64, 8 x mean))
 * run the vector-lane kernel with VL = pow2floor(mean / 6) in [1, 8]: fp64 and
 * integer rows as the emitted TeamPolicy mapping (shuffle-tree reduce, the
 * Kokkos ThreadVectorRange semantics), fp32 rows — and every dtype once
 * lapis_b200_csr_plan_set_exact(plan, 1) — folded in the reference's
 * sequential order (bit-identical).  Irregular structures with a monotone
 * rowptr run the warp-block kernel (blocks of 32 rows handed out dynamically,
 * their contiguous entry range streamed with coalesced loads, each row folded
 * in ascending order by its lane; rows longer than 512 entries folded by the
 * whole warp as a fixed tree unless exact mode or fp32); other irregular
 * structures run the row-stream tile kernel (bit-identical for rows <= 512).
 * LAPIS_B200_SPMV_KERNEL = wb / vec / tile forces a kernel (tuning runs). */
int lapis_b200_csr_plan_info(lapis_b200_csr_plan plan, int64_t* out4);
int lapis_b200_csr_plan_set_exact(lapis_b200_csr_plan plan, int exact);

/* Row-block-sharded SpMV over NCCL (SURVEY 8(b) "sharded spmv_csr_rowblock with
 * an ncclComm_t", 8(e); the native counterpart of sharded.py's RowBlockSpmv).
 * Rank `rank` of `world` owns the global rows [row_begins[rank],
 * row_begins[rank+1]) (row_begins has world + 1 entries); its rowptr is the
 * shard's, rebased to 0, colind holds GLOBAL column indices, x_full is indexed by
 * global column with this rank's slice in place.  Creation (synchronous,
 * collective over `comm`) finds, per owner, the interval of columns the shard
 * reads, all-gathers those intervals and splits the shard at the longest run
 * of rows with only local columns.  Each multiply moves exactly the needed x
 * slabs with ncclSend/ncclRecv on a private stream, overlapped with the
 * interior rows, then multiplies the boundary rows: results are bit-identical
 * to the unsharded multiply.  comm may be NULL when world == 1.
 * The communicator: lapis_b200_nccl_unique_id on one rank, broadcast its 128
 * bytes, lapis_b200_nccl_comm_init on every rank (NCCL is dlopen'ed).
 * rowblock_info: out[0..1] = interior run [a, b); then per peer p
 * out[2+4p .. 5+4p] = needs lo, hi, sends lo, hi. */
typedef struct lapis_b200_rowblock_s* lapis_b200_rowblock;
int lapis_b200_nccl_unique_id(void* out128);
int lapis_b200_nccl_comm_init(const void* id128, int world, int rank, void** out_comm);
int lapis_b200_nccl_comm_destroy(void* comm);
int lapis_b200_rowblock_create(void* comm, int rank, int world, const int64_t* row_begins,
                               const void* rowptr, int rowptr_bytes, const void* colind,
                               int colind_bytes, int64_t nnz, int exact, void* stream,
                               lapis_b200_rowblock* out);
int lapis_b200_rowblock_info(lapis_b200_rowblock rb, int64_t* out);
int lapis_b200_spmv_csr_rowblock(lapis_b200_rowblock rb, const void* rowptr, int rowptr_bytes,
                                 const void* colind, int colind_bytes, const void* values,
                                 void* x_full, void* y_local, int dtype, void* stream);
int lapis_b200_rowblock_destroy(lapis_b200_rowblock rb);

/* Structure validation (synchronous: reads two flags back).  The reference
 * interpreter bounds-checks every load (interp.py:269-276); the tuned kernels
 * do not, so the executor validates a CSR once before using them.
 * out4[0] = 0 ok, 1 a row range leaves [0, nentries), 2 a column leaves
 * [0, ncols), 3 rowptr decreases somewhere (legal: such rows are empty, but
 * the tuned kernels assume monotone rowptr); out4[1] = raw flag bits;
 * out4[3] = rowptr[nrows] - rowptr[0]. */
int lapis_b200_csr_check(int64_t nrows, const void* rowptr, int rowptr_bytes,
                         const void* colind, int colind_bytes, int64_t nentries,
                         int64_t ncols, int64_t* out4, void* stream);

/* ------------------------------------------------------------- CSR x dense SpMM
 * Y[i, c] = sum_j values[j] * X[colind[j], c],  c in [0, k)
 * No reference op: replaces the emitted loop-nest kernel of
 * oracle/ir/spmm.mlir (thread_parallel over N*K, same per-(i, c) order as
 * interp.py:798-812).  Rows with <= 4096 entries are summed sequentially per
 * column (bit-identical); longer rows are split and combined in fixed order. */
int lapis_b200_spmm_csr(int64_t nrows, int64_t ncols, int64_t nnz, int64_t k,
                        const void* rowptr, int rowptr_bytes,
                        const void* colind, int colind_bytes,
                        const void* values, const void* X, int64_t ldx,
                        void* Y, int64_t ldy, int dtype, void* stream);

/* ------------------------------------------------------------------ dense
 * C = A * B — LAPIS::gemm (runtime_header.py:249-266, emitted by
 * emitter.py:550-552 after linalg_lowering.py:32-45), same math as the loop
 * route linalg.matmul (interp.py:711-722). */
int lapis_b200_gemm(int64_t m, int64_t n, int64_t k,
                    const void* A, int64_t lda, const void* B, int64_t ldb,
                    void* C, int64_t ldc, int dtype, int mode, void* stream);
/* y = A * x — LAPIS::gemv (runtime_header.py:268-282; interp.py:729-739). */
int lapis_b200_gemv(int64_t m, int64_t n, const void* A, int64_t lda,
                    const void* x, void* y, int dtype, void* stream);
/* C[b] = A[b] * B[b], contiguous batches — linalg.batch_matmul
 * (linalg_lowering.py:158-173, interp.py:746-763). */
int lapis_b200_batch_gemm(int64_t batch, int64_t m, int64_t n, int64_t k,
                          const void* A, const void* B, void* C, int dtype, int mode,
                          void* stream);
/* out = fold over one axis of a row-major rows x cols array — linalg.reduce /
 * parallel_reduce (linalg_lowering.py:214-252, interp.py:779-795).
 * axis = 1: out[rows]; axis = 0: out[cols]. */
int lapis_b200_reduce_2d(int64_t rows, int64_t cols, const void* src, void* out,
                         int axis, int combiner, int dtype, void* stream);
/* y = (x > 0) ? x : 0 — linalg.elementwise{cmpf ogt; select} (the GCN ReLU,
 * interp.py:520-545, 766-776). */
int lapis_b200_relu(int64_t n, const void* x, void* y, int dtype, void* stream);

/* ------------------------------------------------------------- SpMM plans
 * Structure-only analysis for repeated Y = A X on one CSR structure with a new
 * dense X every call (config 3, the GCN's features).  The plan counts how
 * often each X row is referenced, keeps a remapped private copy of colind and
 * a buffer for the most referenced rows (hot_bytes: 0 = 16 MB, capped by the
 * device's persisting-L2 limit); every lapis_b200_spmm_csr_plan call copies
 * those rows of X into the buffer, pins it in L2 (persisting access-policy
 * window on the stream for the call) and runs the SpMM with hot rows read from
 * it.  Same results as lapis_b200_spmm_csr (per-row order unchanged).  The
 * caller's rowptr / colind must stay as they were at plan creation. */
typedef void* lapis_b200_spmm_plan;
int lapis_b200_spmm_plan_create(int64_t nrows, int64_t ncols, int64_t nnz, int64_t k,
                                const void* rowptr, int rowptr_bytes, const void* colind,
                                int colind_bytes, int dtype, int64_t hot_bytes, void* stream,
                                lapis_b200_spmm_plan* out);
/* out4 = {hot rows, entries reading a hot row, persisting bytes granted, nnz} */
int lapis_b200_spmm_plan_info(lapis_b200_spmm_plan plan, int64_t* out4);
/* *out_far = entries carrying the plan's far-reuse hint (loaded L2 evict_first:
 * the X row's next use lies beyond the plan's reuse horizon), -1 when the plan
 * has no hints. */
int lapis_b200_spmm_plan_hints(lapis_b200_spmm_plan plan, int64_t* out_far);
int lapis_b200_spmm_plan_destroy(lapis_b200_spmm_plan plan);
int lapis_b200_spmm_csr_plan(lapis_b200_spmm_plan plan, const void* rowptr, int rowptr_bytes,
                             const void* colind, int colind_bytes, const void* values,
                             const void* X, int64_t ldx, void* Y, int64_t ldy, int dtype,
                             void* stream);

/* ---------------------------------------------------------------- GCN layer
 * H = relu((A_hat X) W): config 4, the reference's one-function GCN
 * (oracle/ir/gcn_f32.mlir: loop-nest SpMM + linalg.matmul + linalg.elementwise
 * cmpf ogt / select).  X is [ncols, fin], W [fin, fout], H
 * [nrows, fout], row-major.  The SpMM stage always sums in the reference's
 * order; the dense stage (A_hat X) W + ReLU runs on the tcgen05 tensor cores
 * (3xTF32, within the 1e-5 fp32 contract) for fp32 with fin = 64 and
 * fout in {32, 64}, else in the reference order.  dtype F32 or F64. */
int lapis_b200_gcn_layer(int64_t nrows, int64_t ncols, int64_t nnz,
                         const void* rowptr, int rowptr_bytes,
                         const void* colind, int colind_bytes, const void* values,
                         const void* X, int64_t fin, const void* W, int64_t fout, void* H,
                         int dtype, void* stream);
/* The same with the dense stage's mode: LAPIS_B200_GEMM_AUTO (as above) or
 * LAPIS_B200_GEMM_EXACT (reference order for both stages: bit-identical to
 * the reference interpreter). */
int lapis_b200_gcn_layer_mode(int64_t nrows, int64_t ncols, int64_t nnz,
                              const void* rowptr, int rowptr_bytes,
                              const void* colind, int colind_bytes, const void* values,
                              const void* X, int64_t fin, const void* W, int64_t fout, void* H,
                              int mode, int dtype, void* stream);

/* ------------------------------------------------------- synthetic inputs
 * Not reference interfaces: on-device generators for the benchmark matrices
 * (SURVEY 8(d)), rows [row_begin, row_end) of an n^d-point grid, natural
 * ordering, sorted columns.  points = 5 (2-D, diag 4, off -1) or 27 (3-D,
 * diag 26, off -1).  rowptr (int64, row_end-row_begin+1 entries) is rebased to
 * 0; colind (int32) holds global columns.  Pass colind = values = NULL to
 * fill rowptr only. */
int lapis_b200_synth_stencil(int points, int64_t n, int64_t row_begin, int64_t row_end,
                             int64_t* rowptr, int32_t* colind, double* values, void* stream);

/* ------------------------------------------------------- on-disk inputs
 * Matrix Market coordinate files (the paper's SuiteSparse matrices,
 * PAPER.md:349-376) read straight into host CSR, in
 * parallel.  Host-only (no device needed).  mm_info: out4 = {nrows, ncols,
 * nnz after symmetric expansion, flags (bit 0 pattern, bit 1 integer,
 * bits 2-3: 0 general, 1 symmetric, 2 skew-symmetric, 3 hermitian)}.
 * mm_read_csr fills rowptr [nrows + 1] (int64), colind [nnz] (4- or 8-byte),
 * values [nnz] (f64, may be NULL): rows sorted by column, symmetric storage
 * mirrored (skew: negated). */
int lapis_b200_mm_info(const char* path, int64_t* out4);
int lapis_b200_mm_read_csr(const char* path, int64_t* rowptr, void* colind, int colind_bytes,
                           double* values);

/* ------------------------------------------------------- generated kernels
 * The reference turns every kokkos.{range,thread,team}_parallel nest into a
 * Kokkos parallel_for / parallel_reduce lambda (emitter.py:596-780) compiled
 * ahead of time.  Nests with no hand-written kernel above are emitted as CUDA
 * C++ by the executor (paper_2509_25605_b200/cudagen.py: team -> block, thread
 * -> group of vector_length lanes, vector -> lane) and compiled here for
 * sm_100a with NVRTC (--fmad=false: per-op rounding, exact against the
 * reference).  Kernels are cached per (device, source); the handle stays
 * valid for the life of the process.  A generated kernel takes ONE by-value
 * struct parameter of `params_bytes` bytes. */
int lapis_b200_jit_available(void);
int lapis_b200_jit_compile(const char* source, const char* kernel_name, void** out_kernel);
int lapis_b200_jit_launch(void* kernel, int64_t grid_x, int block_x, int smem_bytes,
                          const void* params, int64_t params_bytes, void* stream);
int lapis_b200_jit_cache_size(void);
/* Compile without loading (no device needed); cubin size in *cubin_bytes. */
int lapis_b200_jit_check(const char* source, const char* kernel_name, int64_t* cubin_bytes);

#ifdef __cplusplus
}
#endif

#endif /* LAPIS_B200_H */
