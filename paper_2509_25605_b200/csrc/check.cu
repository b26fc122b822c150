// check.cu — CSR structure validation for the executor's hand-written SpMV /
// SpMM path.  The reference interpreter bounds-checks every load
// (interp.py:269-276): a CSR whose row ranges leave colind / values, or whose
// columns leave x, raises InterpError.  The tuned kernels do not check per
// element, so the executor validates a structure once before handing it to
// them (and hands anything irregular to the generated kernel, which reports
// the interpreter's exact error).  One streaming pass over rowptr and the
// referenced colind range, grid-stride, flags combined with atomicOr.
#include "common.cuh"

namespace lapis_b200 {
namespace {

enum : unsigned { BAD_RANGE = 1u, BAD_COLUMN = 2u, DECREASING = 4u };

template <class RP, class CI>
__global__ void csr_check_kernel(int64_t nrows, const RP* __restrict__ rowptr,
                                 const CI* __restrict__ colind, int64_t nent, int64_t ncols,
                                 unsigned* __restrict__ flags) {
  const int64_t base = (int64_t)rowptr[0];
  const int64_t end = (int64_t)rowptr[nrows];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned f = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nrows; i += stride) {
    const int64_t b = (int64_t)rowptr[i], e = (int64_t)rowptr[i + 1];
    if (e < b) f |= DECREASING;
    else if (e > b && (b < 0 || e > nent)) f |= BAD_RANGE;
  }
  if (end > base && base >= 0 && end <= nent) {
    for (int64_t j = base + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < end; j += stride) {
      const int64_t c = (int64_t)colind[j];
      if (c < 0 || c >= ncols) f |= BAD_COLUMN;
    }
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if (f && (threadIdx.x & 31) == 0) atomicOr(flags, f);
}

template <class RP, class CI>
int launch_check(int64_t nrows, const void* rp, const void* ci, int64_t nent, int64_t ncols,
                 unsigned* flags, cudaStream_t s) {
  const int64_t work = nrows > 0 ? nrows : 1;
  int64_t grid = (work + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (grid > cap) grid = cap;
  csr_check_kernel<RP, CI><<<(unsigned)grid, 256, 0, s>>>(
      nrows, static_cast<const RP*>(rp), static_cast<const CI*>(ci), nent, ncols, flags);
  return check_launch("csr_check_kernel");
}

}  // namespace
}  // namespace lapis_b200

using namespace lapis_b200;

extern "C" int lapis_b200_csr_check(int64_t nrows, const void* rowptr, int rowptr_bytes,
                                    const void* colind, int colind_bytes, int64_t nentries,
                                    int64_t ncols, int64_t* out4, void* stream) {
  if (nrows < 0 || !rowptr || !out4) return fail(LAPIS_B200_ERR_ARG, "csr_check: bad arguments");
  if ((rowptr_bytes != 4 && rowptr_bytes != 8) || (colind_bytes != 4 && colind_bytes != 8))
    return fail(LAPIS_B200_ERR_ARG, "csr_check: index widths must be 4 or 8 bytes");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  keep_pool_memory();
  unsigned* flags = nullptr;
  LB_TRY(check_cuda(cudaMallocAsync(&flags, sizeof(unsigned), s), "csr_check alloc"));
  LB_TRY(check_cuda(cudaMemsetAsync(flags, 0, sizeof(unsigned), s), "csr_check memset"));
  int rc;
  const bool r8 = rowptr_bytes == 8, c8 = colind_bytes == 8;
  if (r8 && c8) rc = launch_check<long long, long long>(nrows, rowptr, colind, nentries, ncols, flags, s);
  else if (r8) rc = launch_check<long long, int>(nrows, rowptr, colind, nentries, ncols, flags, s);
  else if (c8) rc = launch_check<int, long long>(nrows, rowptr, colind, nentries, ncols, flags, s);
  else rc = launch_check<int, int>(nrows, rowptr, colind, nentries, ncols, flags, s);
  unsigned hflags = 0;
  int64_t ends[2] = {0, 0};
  if (rc == LAPIS_B200_OK) {
    rc = check_cuda(cudaMemcpyAsync(&hflags, flags, sizeof(unsigned), cudaMemcpyDeviceToHost, s),
                    "csr_check readback");
  }
  if (rc == LAPIS_B200_OK) {
    if (r8) {
      rc = check_cuda(cudaMemcpyAsync(&ends[0], rowptr, 8, cudaMemcpyDeviceToHost, s), "rowptr[0]");
      if (rc == LAPIS_B200_OK)
        rc = check_cuda(cudaMemcpyAsync(&ends[1], static_cast<const int64_t*>(rowptr) + nrows, 8,
                                        cudaMemcpyDeviceToHost, s), "rowptr[n]");
    } else {
      int32_t e32[2] = {0, 0};
      rc = check_cuda(cudaMemcpyAsync(&e32[0], rowptr, 4, cudaMemcpyDeviceToHost, s), "rowptr[0]");
      if (rc == LAPIS_B200_OK)
        rc = check_cuda(cudaMemcpyAsync(&e32[1], static_cast<const int32_t*>(rowptr) + nrows, 4,
                                        cudaMemcpyDeviceToHost, s), "rowptr[n]");
      if (rc == LAPIS_B200_OK) rc = check_cuda(cudaStreamSynchronize(s), "csr_check sync");
      ends[0] = e32[0];
      ends[1] = e32[1];
    }
  }
  cudaFreeAsync(flags, s);
  if (rc == LAPIS_B200_OK) rc = check_cuda(cudaStreamSynchronize(s), "csr_check sync");
  if (rc != LAPIS_B200_OK) return rc;
  out4[0] = (hflags & BAD_RANGE) ? 1 : (hflags & BAD_COLUMN) ? 2 : (hflags & DECREASING) ? 3 : 0;
  out4[1] = (int64_t)hflags;
  out4[2] = 0;
  out4[3] = ends[1] - ends[0];
  return LAPIS_B200_OK;
}
