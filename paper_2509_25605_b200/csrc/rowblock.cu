// rowblock.cu — row-block-sharded CSR SpMV over NCCL, native.
//
// The C-ABI counterpart of paper_2509_25605_b200/sharded.py's RowBlockSpmv for
// hosts that do not run Python (the emitted C++, a cgo / JNI binding): rank r
// of `world` owns the global rows [row_begins[r], row_begins[r+1]) — rowptr
// rebased to 0, colind GLOBAL — and x_full is indexed by global
// column with this rank's slice already in place.  The only exchange step of
// the path is x:
//
//   create:   per owner p, the [lo, hi) interval of the columns this shard
//             reads from p's rows (one device pass with 64-bit atomics),
//             all-gathered over NCCL so every rank also knows what it sends;
//             the longest run of local rows whose columns are all owned
//             locally (the interior) splits the shard into three row pieces,
//             each with its own CSR plan (spmv.cu);
//   multiply: the halo slabs move with ncclSend / ncclRecv (one group) on a
//             private communication stream while the interior rows are
//             multiplied on the caller's stream; the boundary pieces follow
//             once the slabs have landed (event wait, no host sync).
//
// Rows are never split, so every y entry is the reference's ascending row sum
// (interp.py:798-812) — bit-identical to the single-GPU multiply.
//
// NCCL is resolved with dlopen("libnccl.so.2") on first use (the same library
// torch.distributed loaded, when it did), so the backend does not link NCCL.
#include "common.cuh"

#include <dlfcn.h>
#include <nccl.h>

#include <climits>
#include <cstring>
#include <mutex>
#include <vector>

namespace lapis_b200 {

int csr_plan_create(int64_t, int64_t, const void*, int, cudaStream_t, void**);
int csr_plan_destroy(void*);
int csr_plan_set_exact(void*, int);
int spmv_csr_plan(void*, const void*, int, const void*, int, const void*, const void*, void*, int,
                  cudaStream_t);

// ------------------------------------------------------------------ NCCL api
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string why;
};

static NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    for (const char* n : {"libnccl.so.2", "libnccl.so"})
      if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL)) != nullptr) break;
    if (!h) {
      api.why = "libnccl.so.2 not found";
      return;
    }
#define LB_SYM(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, "nccl" #f))
    LB_SYM(GetUniqueId); LB_SYM(CommInitRank); LB_SYM(CommDestroy); LB_SYM(Send); LB_SYM(Recv);
    LB_SYM(AllGather); LB_SYM(GroupStart); LB_SYM(GroupEnd); LB_SYM(GetErrorString);
#undef LB_SYM
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv &&
             api.AllGather && api.GroupStart && api.GroupEnd && api.GetErrorString;
    if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
  });
  return api;
}

static int nccl_ready() {
  NcclApi& a = nccl();
  return a.ok ? LAPIS_B200_OK : fail(LAPIS_B200_ERR_UNSUPPORTED, "nccl: " + a.why);
}

static int check_nccl(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return LAPIS_B200_OK;
  return fail(LAPIS_B200_ERR_CUDA, std::string(what) + ": " + nccl().GetErrorString(r));
}

static bool nccl_type(int dtype, ncclDataType_t* t) {
  switch (dtype) {
    case LAPIS_B200_F64: *t = ncclFloat64; return true;
    case LAPIS_B200_F32: *t = ncclFloat32; return true;
    case LAPIS_B200_I64: *t = ncclInt64; return true;
    case LAPIS_B200_I32: *t = ncclInt32; return true;
  }
  return false;
}

// ------------------------------------------------------------- plan kernels
constexpr int RB_MAX_WORLD = 64;

// per owner p: [lo, hi) of the referenced global columns that p owns
template <class CI>
__global__ void rb_column_needs_kernel(int64_t nnz, const CI* __restrict__ colind, int world,
                                       const int64_t* __restrict__ begins,
                                       long long* __restrict__ lohi) {
  __shared__ int64_t b[RB_MAX_WORLD + 1];
  __shared__ long long slo[RB_MAX_WORLD], shi[RB_MAX_WORLD];
  for (int i = threadIdx.x; i <= world; i += blockDim.x) b[i] = begins[i];
  for (int i = threadIdx.x; i < world; i += blockDim.x) {
    slo[i] = LLONG_MAX;
    shi[i] = LLONG_MIN;
  }
  __syncthreads();
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nnz;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = (int64_t)colind[j];
    int lo = 0, hi = world;  // owner: b[p] <= c < b[p+1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (b[mid] <= c) lo = mid; else hi = mid;
    }
    atomicMin(&slo[lo], (long long)c);
    atomicMax(&shi[lo], (long long)c + 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < world; i += blockDim.x) {
    if (slo[i] != LLONG_MAX) atomicMin(&lohi[2 * i], slo[i]);
    if (shi[i] != LLONG_MIN) atomicMax(&lohi[2 * i + 1], shi[i]);
  }
}

__global__ void rb_init_lohi_kernel(int world, long long* lohi) {
  const int i = threadIdx.x;
  if (i < world) {
    lohi[2 * i] = LLONG_MAX;
    lohi[2 * i + 1] = LLONG_MIN;
  }
}

// flag[r] = 1 when local row r reads a column outside [own_lo, own_hi)
template <class RP, class CI>
__global__ void rb_remote_rows_kernel(int64_t nloc, const RP* __restrict__ rowptr,
                                      const CI* __restrict__ colind, int64_t own_lo,
                                      int64_t own_hi, uint8_t* __restrict__ flag) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nloc;
       r += (int64_t)gridDim.x * blockDim.x) {
    uint8_t f = 0;
    for (int64_t j = (int64_t)rowptr[r]; j < (int64_t)rowptr[r + 1]; ++j) {
      const int64_t c = (int64_t)colind[j];
      f |= (c < own_lo || c >= own_hi);
    }
    flag[r] = f;
  }
}

struct RowBlockImpl {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1, device = 0;
  int64_t row_begin = 0, row_end = 0;
  std::vector<int64_t> begins;
  std::vector<int64_t> need_lo, need_hi, send_lo, send_hi;
  int64_t a = 0, b = 0;              // interior run [a, b) of local rows
  void* plans[3] = {nullptr, nullptr, nullptr};  // [0, a), [a, b), [b, nloc)
  int64_t lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_start = nullptr, ev_done = nullptr;
};

static void rb_free(RowBlockImpl* h) {
  if (!h) return;
  for (void* p : h->plans)
    if (p) csr_plan_destroy(p);
  if (h->ev_start) cudaEventDestroy(h->ev_start);
  if (h->ev_done) cudaEventDestroy(h->ev_done);
  if (h->comm_stream) cudaStreamDestroy(h->comm_stream);
  delete h;
}

template <class RP, class CI>
static int rb_analyse(RowBlockImpl* h, const void* rowptr, const void* colind, int64_t nnz,
                      cudaStream_t st) {
  const int64_t nloc = h->row_end - h->row_begin;
  const int W = h->world;
  // 1. column intervals per owner
  int64_t* d_begins = nullptr;
  long long* d_lohi = nullptr;
  long long* d_all = nullptr;
  uint8_t* d_flag = nullptr;
  int rc = check_cuda(cudaMallocAsync((void**)&d_begins, (W + 1) * sizeof(int64_t), st), "alloc(rb)");
  if (rc == LAPIS_B200_OK)
    rc = check_cuda(cudaMallocAsync((void**)&d_lohi, 2 * W * sizeof(long long), st), "alloc(rb)");
  if (rc == LAPIS_B200_OK)
    rc = check_cuda(cudaMallocAsync((void**)&d_all, 2 * W * W * sizeof(long long), st), "alloc(rb)");
  if (rc == LAPIS_B200_OK && nloc > 0)
    rc = check_cuda(cudaMallocAsync((void**)&d_flag, nloc, st), "alloc(rb)");
  if (rc == LAPIS_B200_OK)
    rc = check_cuda(cudaMemcpyAsync(d_begins, h->begins.data(), (W + 1) * sizeof(int64_t),
                                    cudaMemcpyHostToDevice, st), "H2D(rb begins)");
  if (rc == LAPIS_B200_OK) {
    rb_init_lohi_kernel<<<1, RB_MAX_WORLD, 0, st>>>(W, d_lohi);
    if (nnz > 0) {
      const int64_t g = std::min<int64_t>((nnz + 255) / 256, (int64_t)num_sms() * 8);
      rb_column_needs_kernel<CI><<<(unsigned)g, 256, 0, st>>>(nnz, (const CI*)colind, W, d_begins,
                                                               d_lohi);
    }
    rc = check_launch("rb_column_needs_kernel");
  }
  // 2. everyone's needs: all-gather of the [world][2] intervals
  if (rc == LAPIS_B200_OK && W > 1)
    rc = check_nccl(nccl().AllGather(d_lohi, d_all, 2 * W, ncclInt64, h->comm, st),
                    "ncclAllGather(rb needs)");
  // 3. interior run
  if (rc == LAPIS_B200_OK && nloc > 0) {
    const int64_t g = std::min<int64_t>((nloc + 255) / 256, (int64_t)num_sms() * 8);
    rb_remote_rows_kernel<RP, CI><<<(unsigned)g, 256, 0, st>>>(
        nloc, (const RP*)rowptr, (const CI*)colind, h->row_begin, h->row_end, d_flag);
    rc = check_launch("rb_remote_rows_kernel");
  }
  std::vector<long long> mine(2 * W), all(2 * W * W);
  std::vector<uint8_t> flag(nloc);
  if (rc == LAPIS_B200_OK)
    rc = check_cuda(cudaMemcpyAsync(mine.data(), d_lohi, 2 * W * sizeof(long long),
                                    cudaMemcpyDeviceToHost, st), "D2H(rb)");
  if (rc == LAPIS_B200_OK && W > 1)
    rc = check_cuda(cudaMemcpyAsync(all.data(), d_all, 2 * W * W * sizeof(long long),
                                    cudaMemcpyDeviceToHost, st), "D2H(rb)");
  if (rc == LAPIS_B200_OK && nloc > 0)
    rc = check_cuda(cudaMemcpyAsync(flag.data(), d_flag, nloc, cudaMemcpyDeviceToHost, st), "D2H(rb)");
  if (rc == LAPIS_B200_OK) rc = check_cuda(cudaStreamSynchronize(st), "sync(rb)");
  cudaFreeAsync(d_begins, st);
  cudaFreeAsync(d_lohi, st);
  cudaFreeAsync(d_all, st);
  if (d_flag) cudaFreeAsync(d_flag, st);
  if (rc != LAPIS_B200_OK) return rc;
  h->need_lo.assign(W, 0); h->need_hi.assign(W, 0);
  h->send_lo.assign(W, 0); h->send_hi.assign(W, 0);
  for (int p = 0; p < W; ++p) {
    if (mine[2 * p] < mine[2 * p + 1]) {
      h->need_lo[p] = mine[2 * p];
      h->need_hi[p] = mine[2 * p + 1];
    }
    if (W > 1) {
      // peer p's needs from this rank
      const long long l = all[(size_t)p * 2 * W + 2 * h->rank];
      const long long u = all[(size_t)p * 2 * W + 2 * h->rank + 1];
      if (l < u) {
        h->send_lo[p] = l;
        h->send_hi[p] = u;
      }
    }
  }
  // longest run of rows without a remote column (sharded.interior_run)
  int64_t best_a = 0, best_len = 0, run = 0;
  for (int64_t r = 0; r <= nloc; ++r) {
    if (r < nloc && !flag[r]) { ++run; continue; }
    if (run > best_len) { best_len = run; best_a = r - run; }
    run = 0;
  }
  h->a = W > 1 ? best_a : 0;
  h->b = W > 1 ? best_a + best_len : nloc;
  return LAPIS_B200_OK;
}

template <class RP>
static int rb_dispatch_ci(RowBlockImpl* h, const void* rp, const void* ci, int ci_bytes,
                          int64_t nnz, cudaStream_t st) {
  return ci_bytes == 8 ? rb_analyse<RP, int64_t>(h, rp, ci, nnz, st)
                       : rb_analyse<RP, int32_t>(h, rp, ci, nnz, st);
}

}  // namespace lapis_b200

using namespace lapis_b200;

extern "C" {

int lapis_b200_nccl_unique_id(void* out128) {
  LB_TRY(nccl_ready());
  if (!out128) return fail(LAPIS_B200_ERR_ARG, "nccl_unique_id: null out");
  ncclUniqueId id;
  LB_TRY(check_nccl(nccl().GetUniqueId(&id), "ncclGetUniqueId"));
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  memcpy(out128, &id, sizeof(id));
  return LAPIS_B200_OK;
}

int lapis_b200_nccl_comm_init(const void* id128, int world, int rank, void** out_comm) {
  LB_TRY(nccl_ready());
  if (!id128 || !out_comm || world < 1 || rank < 0 || rank >= world)
    return fail(LAPIS_B200_ERR_ARG, "nccl_comm_init: bad arguments");
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  ncclComm_t c = nullptr;
  LB_TRY(check_nccl(nccl().CommInitRank(&c, world, id, rank), "ncclCommInitRank"));
  *out_comm = c;
  return LAPIS_B200_OK;
}

int lapis_b200_nccl_comm_destroy(void* comm) {
  if (!comm) return LAPIS_B200_OK;
  LB_TRY(nccl_ready());
  return check_nccl(nccl().CommDestroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
}

int lapis_b200_rowblock_create(void* comm, int rank, int world, const int64_t* row_begins,
                               const void* rowptr, int rowptr_bytes, const void* colind,
                               int colind_bytes, int64_t nnz, int exact, void* stream,
                               lapis_b200_rowblock* out) {
  LB_RANGE("lapis_b200_rowblock_create");
  if (!out) return fail(LAPIS_B200_ERR_ARG, "rowblock_create: null out");
  *out = nullptr;
  if (world < 1 || world > RB_MAX_WORLD || rank < 0 || rank >= world || !row_begins || !rowptr ||
      (rowptr_bytes != 4 && rowptr_bytes != 8) || (colind_bytes != 4 && colind_bytes != 8) ||
      nnz < 0 || (nnz > 0 && !colind))
    return fail(LAPIS_B200_ERR_ARG, "rowblock_create: bad arguments");
  if (world > 1 && !comm) return fail(LAPIS_B200_ERR_ARG, "rowblock_create: null comm");
  for (int p = 0; p < world; ++p)
    if (row_begins[p + 1] < row_begins[p])
      return fail(LAPIS_B200_ERR_ARG, "rowblock_create: row_begins must be non-decreasing");
  if (world > 1) LB_TRY(nccl_ready());
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  auto* h = new RowBlockImpl();
  h->comm = static_cast<ncclComm_t>(comm);
  h->rank = rank;
  h->world = world;
  cudaGetDevice(&h->device);
  h->begins.assign(row_begins, row_begins + world + 1);
  h->row_begin = row_begins[rank];
  h->row_end = row_begins[rank + 1];
  const int64_t nloc = h->row_end - h->row_begin;
  int64_t rp0 = 0;  // the shard's rowptr must be rebased: colind[0] is its first entry
  int rc = check_cuda(cudaMemcpy(&rp0, rowptr, rowptr_bytes, cudaMemcpyDeviceToHost), "D2H(rb rowptr)");
  if (rowptr_bytes == 4) rp0 = (int32_t)(rp0 & 0xffffffffLL);
  if (rc == LAPIS_B200_OK && rp0 != 0)
    rc = fail(LAPIS_B200_ERR_ARG, "rowblock_create: the shard's rowptr must start at 0");
  if (rc != LAPIS_B200_OK) {
    rb_free(h);
    return rc;
  }
  rc = rowptr_bytes == 8 ? rb_dispatch_ci<int64_t>(h, rowptr, colind, colind_bytes, nnz, st)
                             : rb_dispatch_ci<int32_t>(h, rowptr, colind, colind_bytes, nnz, st);
  const int64_t cuts[4] = {0, h->a, h->b, nloc};
  int64_t rpv[4] = {0, 0, 0, 0};  // rowptr at the cuts: each piece's nonzero count
  for (int i = 0; i < 4 && rc == LAPIS_B200_OK; ++i) {
    const char* src = static_cast<const char*>(rowptr) + cuts[i] * rowptr_bytes;
    if (rowptr_bytes == 8) {
      rc = check_cuda(cudaMemcpy(&rpv[i], src, 8, cudaMemcpyDeviceToHost), "D2H(rb rowptr)");
    } else {
      int32_t v = 0;
      rc = check_cuda(cudaMemcpy(&v, src, 4, cudaMemcpyDeviceToHost), "D2H(rb rowptr)");
      rpv[i] = v;
    }
  }
  for (int i = 0; i < 3 && rc == LAPIS_B200_OK; ++i) {
    h->lo[i] = cuts[i];
    h->hi[i] = cuts[i + 1];
    if (h->hi[i] <= h->lo[i]) continue;
    const char* base = static_cast<const char*>(rowptr) + h->lo[i] * rowptr_bytes;
    const int64_t pnnz = rpv[i + 1] > rpv[i] ? rpv[i + 1] - rpv[i] : 0;
    rc = csr_plan_create(h->hi[i] - h->lo[i], pnnz, base, rowptr_bytes, st, &h->plans[i]);
    if (rc == LAPIS_B200_OK && exact) rc = csr_plan_set_exact(h->plans[i], 1);
  }
  if (rc == LAPIS_B200_OK && world > 1) {
    rc = check_cuda(cudaStreamCreateWithFlags(&h->comm_stream, cudaStreamNonBlocking), "stream(rb)");
    if (rc == LAPIS_B200_OK)
      rc = check_cuda(cudaEventCreateWithFlags(&h->ev_start, cudaEventDisableTiming), "event(rb)");
    if (rc == LAPIS_B200_OK)
      rc = check_cuda(cudaEventCreateWithFlags(&h->ev_done, cudaEventDisableTiming), "event(rb)");
  }
  if (rc != LAPIS_B200_OK) {
    rb_free(h);
    return rc;
  }
  *out = reinterpret_cast<lapis_b200_rowblock>(h);
  return LAPIS_B200_OK;
}

int lapis_b200_rowblock_info(lapis_b200_rowblock handle, int64_t* out) {
  auto* h = reinterpret_cast<RowBlockImpl*>(handle);
  if (!h || !out) return fail(LAPIS_B200_ERR_ARG, "rowblock_info: null argument");
  out[0] = h->a;
  out[1] = h->b;
  for (int p = 0; p < h->world; ++p) {
    out[2 + 4 * p] = h->need_lo[p];
    out[3 + 4 * p] = h->need_hi[p];
    out[4 + 4 * p] = h->send_lo[p];
    out[5 + 4 * p] = h->send_hi[p];
  }
  return LAPIS_B200_OK;
}

int lapis_b200_spmv_csr_rowblock(lapis_b200_rowblock handle, const void* rowptr, int rowptr_bytes,
                                 const void* colind, int colind_bytes, const void* values,
                                 void* x_full, void* y_local, int dtype, void* stream) {
  LB_RANGE("lapis_b200_spmv_csr_rowblock");
  auto* h = reinterpret_cast<RowBlockImpl*>(handle);
  if (!h) return fail(LAPIS_B200_ERR_ARG, "spmv_rowblock: null handle");
  if (!valid_dtype(dtype)) return fail(LAPIS_B200_ERR_ARG, "spmv_rowblock: unsupported dtype");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const size_t es = (size_t)elem_bytes(dtype);
  auto piece = [&](int i) -> int {
    if (!h->plans[i]) return LAPIS_B200_OK;
    const char* rp = static_cast<const char*>(rowptr) + h->lo[i] * rowptr_bytes;
    char* y = static_cast<char*>(y_local) + h->lo[i] * es;
    return spmv_csr_plan(h->plans[i], rp, rowptr_bytes, colind, colind_bytes, values, x_full, y,
                         dtype, st);
  };
  if (h->world == 1) return piece(1);
  ncclDataType_t t;
  if (!nccl_type(dtype, &t)) return fail(LAPIS_B200_ERR_ARG, "spmv_rowblock: dtype");
  // halo slabs on the communication stream, ordered after the caller's work
  LB_TRY(check_cuda(cudaEventRecord(h->ev_start, st), "event(rb start)"));
  LB_TRY(check_cuda(cudaStreamWaitEvent(h->comm_stream, h->ev_start, 0), "wait(rb start)"));
  LB_TRY(check_nccl(nccl().GroupStart(), "ncclGroupStart"));
  int rc = LAPIS_B200_OK;
  char* xb = static_cast<char*>(x_full);
  for (int p = 0; p < h->world && rc == LAPIS_B200_OK; ++p) {
    if (p == h->rank) continue;
    if (h->send_hi[p] > h->send_lo[p])
      rc = check_nccl(nccl().Send(xb + h->send_lo[p] * es, (size_t)(h->send_hi[p] - h->send_lo[p]),
                                  t, p, h->comm, h->comm_stream), "ncclSend");
    if (rc == LAPIS_B200_OK && h->need_hi[p] > h->need_lo[p])
      rc = check_nccl(nccl().Recv(xb + h->need_lo[p] * es, (size_t)(h->need_hi[p] - h->need_lo[p]),
                                  t, p, h->comm, h->comm_stream), "ncclRecv");
  }
  const int rg = check_nccl(nccl().GroupEnd(), "ncclGroupEnd");
  if (rc == LAPIS_B200_OK) rc = rg;
  if (rc == LAPIS_B200_OK)
    rc = check_cuda(cudaEventRecord(h->ev_done, h->comm_stream), "event(rb done)");
  if (rc == LAPIS_B200_OK) rc = piece(1);  // interior rows while the slabs move
  if (rc == LAPIS_B200_OK)
    rc = check_cuda(cudaStreamWaitEvent(st, h->ev_done, 0), "wait(rb done)");
  if (rc == LAPIS_B200_OK) rc = piece(0);
  if (rc == LAPIS_B200_OK) rc = piece(2);
  return rc;
}

int lapis_b200_rowblock_destroy(lapis_b200_rowblock handle) {
  rb_free(reinterpret_cast<RowBlockImpl*>(handle));
  return LAPIS_B200_OK;
}

}  // extern "C"
