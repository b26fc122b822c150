// gcn.cu — the config-4 GCN layer H = relu((A_hat X) W) as one library call.
//
// The reference expresses it as one IR function (oracle/ir/gcn_f32.mlir,
// SURVEY A.5): a loop-nest SpMM into a device-local temporary, linalg.matmul
// into a second temporary, and linalg.elementwise ReLU (cmpf ogt + select).
// Here: the SpMM kernels (reference order per output column, fp32 hub rows
// included) write A_hat X to a stream-ordered workspace, then the dense stage
// applies W with the ReLU select fused into its store: on the tcgen05 tensor
// cores (gcn_dense.cu, 3xTF32, within the 1e-5 fp32 contract) in AUTO mode,
// or in the reference's summation order (EXACT mode: H bit-identical to the
// reference interpreter, tests/test_gcn_gpu.py).
//
// Optionally (LAPIS_B200_GCN_FUSED=1; fp32, fin = fout = 64) FUSED: the SpMM batch
// kernel applies W (shared memory) and the ReLU to each row as soon as the
// row's 64 sums are complete and writes only H — no A_hat X round trip through
// HBM and one pass over A; hub rows (> 2048 entries) are folded into H by the
// exact long-row kernel and finished in place by a per-row epilogue kernel.
// Same arithmetic in the same order, so still bit-identical.
#include "common.cuh"

#include <cstdlib>

namespace lapis_b200 {

int spmm_csr(int64_t, int64_t, int64_t, int64_t, const void*, int, const void*, int, const void*,
             const void*, int64_t, void*, int64_t, int, cudaStream_t);
int gemm_exact_relu(int64_t, int64_t, int64_t, const void*, int64_t, const void*, int64_t, void*,
                    int64_t, int, cudaStream_t);
int spmm_gcn_fused(int64_t, int64_t, const void*, int, const void*, int, const void*, const void*,
                   int64_t, const void*, void*, int64_t, cudaStream_t);
bool gcn_dense_tc_ok(int64_t, int64_t, int64_t, const void*, int64_t, const void*, int64_t);
int gcn_dense_tf32x3(int64_t, int64_t, int64_t, const void*, int64_t, const void*, int64_t, void*,
                     int64_t, cudaStream_t);

// the fused single-pass path (LAPIS_B200_GCN_FUSED=1): fp32, fin = fout = 64,
// 8-byte aligned X / H rows.  Not the default: measured on B200 (config 4) the
// fused batch kernel took 1.76 ms against 1.16 ms SpMM + 0.52 ms GEMM — the
// per-row epilogue (64 shuffles + 64 shared loads + 256 separately rounded
// mul/add per lane) stalls the warp's gather pipeline, which costs more than
// the 512 MB A_hat X round trip it saves
static bool gcn_fusable(int dtype, int64_t fin, int64_t fout, const void* X, const void* H) {
  const char* e = getenv("LAPIS_B200_GCN_FUSED");
  const bool on = e && e[0] == '1';
  return on && dtype == LAPIS_B200_F32 && fin == 64 && fout == 64 &&
         (uintptr_t)X % 8 == 0 && (uintptr_t)H % 8 == 0;
}

int gcn_layer(int64_t nrows, int64_t ncols, int64_t nnz, const void* rowptr, int rp_bytes,
              const void* colind, int ci_bytes, const void* values, const void* X, int64_t fin,
              const void* W, int64_t fout, void* H, int mode, int dtype, cudaStream_t st) {
  if (dtype != LAPIS_B200_F32 && dtype != LAPIS_B200_F64)
    return fail(LAPIS_B200_ERR_UNSUPPORTED, "gcn: floating-point dtypes only");
  if (nrows < 0 || fin < 0 || fout < 0) return fail(LAPIS_B200_ERR_ARG, "gcn: negative extent");
  if (nrows == 0 || fout == 0) return LAPIS_B200_OK;
  if (!W || !H) return fail(LAPIS_B200_ERR_ARG, "gcn: null operand");
  if (mode == LAPIS_B200_GEMM_EXACT && gcn_fusable(dtype, fin, fout, X, H))
    return spmm_gcn_fused(nrows, nnz, rowptr, rp_bytes, colind, ci_bytes, values, X, fin, W, H,
                          fout, st);
  const size_t es = (size_t)elem_bytes(dtype);
  void* ax = nullptr;
  LB_TRY(check_cuda(cudaMallocAsync(&ax, (size_t)nrows * (size_t)(fin > 0 ? fin : 1) * es, st),
                    "alloc(gcn A_hat X)"));
  int rc = LAPIS_B200_OK;
  if (fin > 0)
    rc = spmm_csr(nrows, ncols, nnz, fin, rowptr, rp_bytes, colind, ci_bytes, values, X, fin, ax,
                  fin, dtype, st);
  if (rc == LAPIS_B200_OK) {
    // dense stage: tcgen05 3xTF32 + fused ReLU (AUTO, fp32, fin 64, fout 32 / 64),
    // else the reference-order kernel (EXACT: bit-identical)
    if (mode == LAPIS_B200_GEMM_AUTO && dtype == LAPIS_B200_F32 &&
        gcn_dense_tc_ok(nrows, fout, fin, ax, fin, H, fout))
      rc = gcn_dense_tf32x3(nrows, fout, fin, ax, fin, W, fout, H, fout, st);
    else
      rc = gemm_exact_relu(nrows, fout, fin, ax, fin, W, fout, H, fout, dtype, st);
  }
  cudaFreeAsync(ax, st);
  return rc;
}

}  // namespace lapis_b200
