// capi.cu — the extern "C" boundary declared in include/lapis_b200.h.
// Thin: argument checks, stream casts, error capture; the kernels live in the
// other translation units.
#include "common.cuh"

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include <cstdio>
#include <cstring>

namespace lapis_b200 {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}

int check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return LAPIS_B200_OK;
  const int code = (e == cudaErrorMemoryAllocation) ? LAPIS_B200_ERR_NOMEM : LAPIS_B200_ERR_CUDA;
  return fail(code, std::string(what) + ": " + cudaGetErrorString(e));
}

int check_launch(const char* what) { return check_cuda(cudaGetLastError(), what); }

// kernels (other translation units)
int spmv_csr(int64_t, int64_t, int64_t, const void*, int, const void*, int, const void*,
             const void*, void*, int, int, cudaStream_t);
int csr_plan_create(int64_t, int64_t, const void*, int, cudaStream_t, void**);
int csr_plan_destroy(void*);
int csr_plan_info(void*, int64_t*);
int csr_plan_set_exact(void*, int);
int spmv_csr_plan(void*, const void*, int, const void*, int, const void*, const void*, void*, int,
                  cudaStream_t);
int spmm_csr(int64_t, int64_t, int64_t, int64_t, const void*, int, const void*, int, const void*,
             const void*, int64_t, void*, int64_t, int, cudaStream_t);
int gemm_dispatch(int64_t, int64_t, int64_t, int64_t, const void*, int64_t, const void*, int64_t,
                  void*, int64_t, int64_t, int64_t, int64_t, int, int, cudaStream_t);
int gemv(int64_t, int64_t, const void*, int64_t, const void*, void*, int, cudaStream_t);
int reduce_2d(int64_t, int64_t, const void*, void*, int, int, int, cudaStream_t);
int relu(int64_t, const void*, void*, int, cudaStream_t);
int gcn_layer(int64_t, int64_t, int64_t, const void*, int, const void*, int, const void*,
              const void*, int64_t, const void*, int64_t, void*, int, int, cudaStream_t);
int synth_stencil(int, int64_t, int64_t, int64_t, int64_t*, int32_t*, double*, cudaStream_t);
int spmm_plan_create(int64_t, int64_t, int64_t, int64_t, const void*, int, const void*, int, int,
                     int64_t, cudaStream_t, void**);
int spmm_plan_info(void*, int64_t*);
int spmm_plan_hints(void*, int64_t*);
int spmm_plan_destroy(void*);
int spmm_csr_plan(void*, const void*, int, const void*, int, const void*, const void*, int64_t,
                  void*, int64_t, int, cudaStream_t);
void release_workspaces();

}  // namespace lapis_b200

using namespace lapis_b200;

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" {

const char* lapis_b200_last_error(void) { return g_last_error.c_str(); }

int lapis_b200_version(void) { return 100; }

int lapis_b200_graph_kernels(void* graph, char* buf, int64_t cap, int64_t* nkernels) {
  // kernel nodes of a captured CUDA graph (one bench step), as
  // "name\n" lines: the launch census of the step, independent of any tracer
  if (!graph || !nkernels) return fail(LAPIS_B200_ERR_ARG, "graph_kernels: null argument");
  cudaGraph_t g = reinterpret_cast<cudaGraph_t>(graph);
  size_t n = 0;
  LB_TRY(check_cuda(cudaGraphGetNodes(g, nullptr, &n), "cudaGraphGetNodes"));
  std::vector<cudaGraphNode_t> nodes(n);
  if (n) LB_TRY(check_cuda(cudaGraphGetNodes(g, nodes.data(), &n), "cudaGraphGetNodes"));
  std::string out;
  int64_t k = 0;
  for (auto nd : nodes) {
    cudaGraphNodeType t;
    LB_TRY(check_cuda(cudaGraphNodeGetType(nd, &t), "cudaGraphNodeGetType"));
    if (t != cudaGraphNodeTypeKernel) continue;
    cudaKernelNodeParams p;
    const char* name = nullptr;
    if (cudaGraphKernelNodeGetParams(nd, &p) == cudaSuccess && p.func)
      cudaFuncGetName(&name, p.func);
    cudaGetLastError();
    out += name ? name : "?";
    out += '\n';
    ++k;
  }
  *nkernels = k;
  if (buf && cap > 0) {
    const size_t m = std::min<size_t>(out.size(), (size_t)cap - 1);
    memcpy(buf, out.data(), m);
    buf[m] = 0;
  }
  return LAPIS_B200_OK;
}

int lapis_b200_init(int device) {
  int n = 0;
  LB_TRY(check_cuda(cudaGetDeviceCount(&n), "cudaGetDeviceCount"));
  if (device < 0 || device >= n) return fail(LAPIS_B200_ERR_ARG, "init: no such device");
  LB_TRY(check_cuda(cudaSetDevice(device), "cudaSetDevice"));
  cudaDeviceProp prop;
  LB_TRY(check_cuda(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties"));
  if (prop.major != 10)
    return fail(LAPIS_B200_ERR_UNSUPPORTED, "init: kernels are built for sm_100a (B200)");
  LB_TRY(check_cuda(cudaFree(nullptr), "context init"));
  keep_pool_memory();
  return LAPIS_B200_OK;
}

int lapis_b200_finalize(void) {
  release_workspaces();
  return LAPIS_B200_OK;
}

int64_t lapis_b200_csr_vector_length(int64_t nrows, int64_t nnz, int64_t cap) {
  // loop_mapping.py:224-246: k = ceildivsi(nnz, max(nrows, 1)); smallest power
  // of two p <= cap/2 with k <= p, else cap
  const int64_t rows = nrows > 1 ? nrows : 1;
  int64_t k = nnz / rows;
  if ((nnz % rows != 0) && ((nnz < 0) == (rows < 0))) k += 1;  // runtime_header.py:75-80
  int64_t acc = cap;
  for (int64_t p = cap / 2; p >= 1; p /= 2)
    if (k <= p) acc = p;
  return acc;
}

int lapis_b200_spmv_csr(int64_t nrows, int64_t ncols, int64_t nnz, const void* rowptr,
                        int rowptr_bytes, const void* colind, int colind_bytes,
                        const void* values, const void* x, void* y, int dtype,
                        int vector_length, void* stream) {
  LB_RANGE("lapis_b200_spmv_csr");
  keep_pool_memory();
  return spmv_csr(nrows, ncols, nnz, rowptr, rowptr_bytes, colind, colind_bytes, values, x, y,
                  dtype, vector_length, S(stream));
}

int lapis_b200_csr_plan_create(int64_t nrows, int64_t nnz, const void* rowptr, int rowptr_bytes,
                               void* stream, lapis_b200_csr_plan* out_plan) {
  LB_RANGE("lapis_b200_csr_plan_create");
  keep_pool_memory();
  return csr_plan_create(nrows, nnz, rowptr, rowptr_bytes, S(stream),
                         reinterpret_cast<void**>(out_plan));
}

int lapis_b200_csr_plan_destroy(lapis_b200_csr_plan plan) { return csr_plan_destroy(plan); }

int lapis_b200_csr_plan_info(lapis_b200_csr_plan plan, int64_t* out4) {
  return csr_plan_info(plan, out4);
}

int lapis_b200_csr_plan_set_exact(lapis_b200_csr_plan plan, int exact) {
  return csr_plan_set_exact(plan, exact);
}

int lapis_b200_spmv_csr_plan(lapis_b200_csr_plan plan, const void* rowptr, int rowptr_bytes,
                             const void* colind, int colind_bytes, const void* values,
                             const void* x, void* y, int dtype, void* stream) {
  LB_RANGE("lapis_b200_spmv_csr_plan");
  return spmv_csr_plan(plan, rowptr, rowptr_bytes, colind, colind_bytes, values, x, y, dtype,
                       S(stream));
}

int lapis_b200_spmm_csr(int64_t nrows, int64_t ncols, int64_t nnz, int64_t k, const void* rowptr,
                        int rowptr_bytes, const void* colind, int colind_bytes,
                        const void* values, const void* X, int64_t ldx, void* Y, int64_t ldy,
                        int dtype, void* stream) {
  LB_RANGE("lapis_b200_spmm_csr");
  keep_pool_memory();
  return spmm_csr(nrows, ncols, nnz, k, rowptr, rowptr_bytes, colind, colind_bytes, values, X,
                  ldx, Y, ldy, dtype, S(stream));
}

int lapis_b200_spmm_plan_create(int64_t nrows, int64_t ncols, int64_t nnz, int64_t k,
                                 const void* rowptr, int rowptr_bytes, const void* colind,
                                 int colind_bytes, int dtype, int64_t hot_bytes, void* stream,
                                 lapis_b200_spmm_plan* out) {
  LB_RANGE("lapis_b200_spmm_plan_create");
  keep_pool_memory();
  return spmm_plan_create(nrows, ncols, nnz, k, rowptr, rowptr_bytes, colind, colind_bytes, dtype,
                          hot_bytes, S(stream), out);
}

int lapis_b200_spmm_plan_info(lapis_b200_spmm_plan plan, int64_t* out4) {
  return spmm_plan_info(plan, out4);
}

int lapis_b200_spmm_plan_hints(lapis_b200_spmm_plan plan, int64_t* out_far) {
  return spmm_plan_hints(plan, out_far);
}

int lapis_b200_spmm_plan_destroy(lapis_b200_spmm_plan plan) { return spmm_plan_destroy(plan); }

int lapis_b200_spmm_csr_plan(lapis_b200_spmm_plan plan, const void* rowptr, int rowptr_bytes,
                             const void* colind, int colind_bytes, const void* values,
                             const void* X, int64_t ldx, void* Y, int64_t ldy, int dtype,
                             void* stream) {
  LB_RANGE("lapis_b200_spmm_csr_plan");
  return spmm_csr_plan(plan, rowptr, rowptr_bytes, colind, colind_bytes, values, X, ldx, Y, ldy,
                       dtype, S(stream));
}

int lapis_b200_gemm(int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B,
                    int64_t ldb, void* C, int64_t ldc, int dtype, int mode, void* stream) {
  LB_RANGE("lapis_b200_gemm");
  keep_pool_memory();
  return gemm_dispatch(1, m, n, k, A, lda, B, ldb, C, ldc, 0, 0, 0, dtype, mode, S(stream));
}

int lapis_b200_gemv(int64_t m, int64_t n, const void* A, int64_t lda, const void* x, void* y,
                    int dtype, void* stream) {
  LB_RANGE("lapis_b200_gemv");
  if (m < 0 || n < 0 || lda < n) return fail(LAPIS_B200_ERR_ARG, "gemv: bad extents");
  if (!valid_dtype(dtype)) return fail(LAPIS_B200_ERR_ARG, "gemv: unsupported dtype");
  if (m > 0 && (!y || (n > 0 && (!A || !x)))) return fail(LAPIS_B200_ERR_ARG, "gemv: null operand");
  return gemv(m, n, A, lda, x, y, dtype, S(stream));
}

int lapis_b200_batch_gemm(int64_t batch, int64_t m, int64_t n, int64_t k, const void* A,
                          const void* B, void* C, int dtype, int mode, void* stream) {
  LB_RANGE("lapis_b200_batch_gemm");
  keep_pool_memory();
  if (batch < 0) return fail(LAPIS_B200_ERR_ARG, "batch_gemm: negative batch");
  return gemm_dispatch(batch, m, n, k, A, k, B, n, C, n, m * k, k * n, m * n, dtype, mode,
                       S(stream));
}

int lapis_b200_reduce_2d(int64_t rows, int64_t cols, const void* src, void* out, int axis,
                         int combiner, int dtype, void* stream) {
  LB_RANGE("lapis_b200_reduce_2d");
  if (rows < 0 || cols < 0) return fail(LAPIS_B200_ERR_ARG, "reduce: negative extent");
  if (!valid_dtype(dtype)) return fail(LAPIS_B200_ERR_ARG, "reduce: unsupported dtype");
  if ((rows > 0 && cols > 0 && !src) || ((axis == 1 ? rows : cols) > 0 && !out))
    return fail(LAPIS_B200_ERR_ARG, "reduce: null operand");
  return reduce_2d(rows, cols, src, out, axis, combiner, dtype, S(stream));
}

int lapis_b200_relu(int64_t n, const void* x, void* y, int dtype, void* stream) {
  LB_RANGE("lapis_b200_relu");
  if (n < 0) return fail(LAPIS_B200_ERR_ARG, "relu: negative extent");
  if (n > 0 && (!x || !y)) return fail(LAPIS_B200_ERR_ARG, "relu: null operand");
  return relu(n, x, y, dtype, S(stream));
}

int lapis_b200_gcn_layer(int64_t nrows, int64_t ncols, int64_t nnz, const void* rowptr,
                         int rowptr_bytes, const void* colind, int colind_bytes, const void* values,
                         const void* X, int64_t fin, const void* W, int64_t fout, void* H,
                         int dtype, void* stream) {
  LB_RANGE("lapis_b200_gcn_layer");
  keep_pool_memory();
  return gcn_layer(nrows, ncols, nnz, rowptr, rowptr_bytes, colind, colind_bytes, values, X, fin,
                   W, fout, H, LAPIS_B200_GEMM_AUTO, dtype, S(stream));
}

int lapis_b200_gcn_layer_mode(int64_t nrows, int64_t ncols, int64_t nnz, const void* rowptr,
                              int rowptr_bytes, const void* colind, int colind_bytes,
                              const void* values, const void* X, int64_t fin, const void* W,
                              int64_t fout, void* H, int mode, int dtype, void* stream) {
  LB_RANGE("lapis_b200_gcn_layer_mode");
  keep_pool_memory();
  if (mode != LAPIS_B200_GEMM_AUTO && mode != LAPIS_B200_GEMM_EXACT)
    return fail(LAPIS_B200_ERR_ARG, "gcn: mode must be AUTO or EXACT");
  return gcn_layer(nrows, ncols, nnz, rowptr, rowptr_bytes, colind, colind_bytes, values, X, fin,
                   W, fout, H, mode, dtype, S(stream));
}

int lapis_b200_synth_stencil(int points, int64_t n, int64_t row_begin, int64_t row_end,
                             int64_t* rowptr, int32_t* colind, double* values, void* stream) {
  LB_RANGE("lapis_b200_synth_stencil");
  keep_pool_memory();
  return synth_stencil(points, n, row_begin, row_end, rowptr, colind, values, S(stream));
}

}  // extern "C"
