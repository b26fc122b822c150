// synth.cu — on-device generators for the benchmark matrices:
// 2-D 5-point and 3-D 27-point stencils on an n^d grid, natural ordering,
// ascending columns, diagonal 4 / 26 and off-diagonals -1.  Not a reference
// interface; these exist so the 5.4e9-nonzero config-5 matrix is built in
// milliseconds on the device instead of minutes on the host.
#include "common.cuh"

namespace lapis_b200 {

// number of in-grid neighbours (including self) of point p along one axis
__device__ __forceinline__ int64_t span(int64_t p, int64_t n) {
  return 1 + (p > 0) + (p < n - 1);
}

// sum_{p < upto} span(p, n), upto in [0, n]
__device__ __forceinline__ int64_t span_prefix(int64_t upto, int64_t n) {
  if (upto <= 0) return 0;
  return upto + (upto - 1) + (upto < n - 1 ? upto : n - 1);
}

// entries before row r (closed form).  5-point: nnz(i,j) = span(i)+span(j)-1;
// 27-point: nnz(i,j,k) = span(i)*span(j)*span(k).
__device__ int64_t nnz_before(int points, int64_t n, int64_t r) {
  const int64_t S = span_prefix(n, n);
  if (points == 5) {
    const int64_t i = r / n, j = r % n;
    return span_prefix(i, n) * n + i * (S - n) + j * span(i, n) + span_prefix(j, n) - j;
  }
  const int64_t n2 = n * n;
  const int64_t i = r / n2, j = (r / n) % n, k = r % n;
  return span_prefix(i, n) * S * S +
         span(i, n) * (span_prefix(j, n) * S + span(j, n) * span_prefix(k, n));
}

__global__ void stencil_rowptr_kernel(int points, int64_t n, int64_t row_begin, int64_t rows,
                                      int64_t base, int64_t* __restrict__ rowptr) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t > rows) return;
  rowptr[t] = nnz_before(points, n, row_begin + t) - base;
}

__global__ void stencil_fill_kernel(int points, int64_t n, int64_t row_begin, int64_t rows,
                                    const int64_t* __restrict__ rowptr,
                                    int32_t* __restrict__ colind, double* __restrict__ values) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= rows) return;
  const int64_t r = row_begin + t;
  int64_t pos = rowptr[t];
  if (points == 5) {
    const int64_t i = r / n, j = r % n;
    const int64_t cols[5] = {r - n, r - 1, r, r + 1, r + n};
    const bool ok[5] = {i > 0, j > 0, true, j < n - 1, i < n - 1};
    for (int q = 0; q < 5; ++q)
      if (ok[q]) { colind[pos] = (int32_t)cols[q]; values[pos] = (q == 2) ? 4.0 : -1.0; ++pos; }
    return;
  }
  const int64_t n2 = n * n;
  const int64_t i = r / n2, j = (r / n) % n, k = r % n;
  for (int di = -1; di <= 1; ++di) {
    if (i + di < 0 || i + di >= n) continue;
    for (int dj = -1; dj <= 1; ++dj) {
      if (j + dj < 0 || j + dj >= n) continue;
      for (int dk = -1; dk <= 1; ++dk) {
        if (k + dk < 0 || k + dk >= n) continue;
        const int64_t col = r + di * n2 + dj * n + dk;
        colind[pos] = (int32_t)col;
        values[pos] = (di == 0 && dj == 0 && dk == 0) ? 26.0 : -1.0;
        ++pos;
      }
    }
  }
}

__global__ void base_kernel(int points, int64_t n, int64_t row_begin, int64_t* out) {
  *out = nnz_before(points, n, row_begin);
}

int synth_stencil(int points, int64_t n, int64_t row_begin, int64_t row_end, int64_t* rowptr,
                  int32_t* colind, double* values, cudaStream_t st) {
  if (points != 5 && points != 27) return fail(LAPIS_B200_ERR_ARG, "synth: points must be 5 or 27");
  const int64_t N = points == 5 ? n * n : n * n * n;
  if (n < 1 || row_begin < 0 || row_end < row_begin || row_end > N || !rowptr)
    return fail(LAPIS_B200_ERR_ARG, "synth: bad row range");
  if (N > 0x7fffffffLL) return fail(LAPIS_B200_ERR_ARG, "synth: grid exceeds int32 columns");
  const int64_t rows = row_end - row_begin;
  int64_t* d_base = nullptr;
  LB_TRY(check_cuda(cudaMallocAsync((void**)&d_base, sizeof(int64_t), st), "cudaMallocAsync"));
  base_kernel<<<1, 1, 0, st>>>(points, n, row_begin, d_base);
  int64_t base = 0;
  LB_TRY(check_cuda(cudaMemcpyAsync(&base, d_base, sizeof(int64_t), cudaMemcpyDeviceToHost, st),
                    "memcpy(base)"));
  LB_TRY(check_cuda(cudaStreamSynchronize(st), "sync(base)"));
  cudaFreeAsync(d_base, st);
  const int threads = 256;
  stencil_rowptr_kernel<<<(unsigned)((rows + 1 + threads - 1) / threads), threads, 0, st>>>(
      points, n, row_begin, rows, base, rowptr);
  LB_TRY(check_launch("stencil_rowptr_kernel"));
  if (colind && values && rows > 0) {
    stencil_fill_kernel<<<(unsigned)((rows + threads - 1) / threads), threads, 0, st>>>(
        points, n, row_begin, rows, rowptr, colind, values);
    LB_TRY(check_launch("stencil_fill_kernel"));
  }
  return LAPIS_B200_OK;
}

}  // namespace lapis_b200
