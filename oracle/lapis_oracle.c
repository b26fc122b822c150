/*
 * lapis_oracle.c — CPU restatement of the LAPIS reference semantics for the
 * hot path (CSR SpMV, CSR x dense SpMM, dense matmul / matvec / batch_matmul,
 * linalg.reduce, the CSR vector-length hint, the GCN ReLU select).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_2509_25605_b200/ links, loads or
 * calls this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg use it, and only as the checker.
 *
 * Semantics follow the reference interpreter (the reference's "semantic
 * oracle", /root/reference/pkg/src/lapis/interp.py): every loop runs
 * sequentially in ascending index order and every arithmetic op is rounded to
 * the element type before the next one (coerce_scalar, interp.py:168-171).
 * The file is compiled with -ffp-contract=off so no multiply-add is fused,
 * which makes it bit-identical to the interpreter (pinned by
 * tests/test_oracle_golden.py against fixtures generated from the reference).
 *
 * Rows are independent, so the row loops may be split over OpenMP threads
 * without changing any per-row summation order.
 *
 * dtype codes (shared with include/lapis_b200.h): 0=f32 1=f64 2=i32 3=i64.
 */
#include <stdint.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { OR_F32 = 0, OR_F64 = 1, OR_I32 = 2, OR_I64 = 3 };

/* integer index load of width 4 or 8 bytes (rowptr / colind may be i32 or
 * i64/index: dialect.py:797-812 accepts both; spmv_lowering.py:15-18 casts) */
static inline int64_t ld_idx(const void* p, int bytes, int64_t i) {
  return bytes == 4 ? (int64_t)((const int32_t*)p)[i] : ((const int64_t*)p)[i];
}

/* wrap-around integer arithmetic (interp.py:145-152 _wrap_int) */
static inline int64_t add_i64(int64_t a, int64_t b) { return (int64_t)((uint64_t)a + (uint64_t)b); }
static inline int64_t mul_i64(int64_t a, int64_t b) { return (int64_t)((uint64_t)a * (uint64_t)b); }
static inline int32_t add_i32(int32_t a, int32_t b) { return (int32_t)((uint32_t)a + (uint32_t)b); }
static inline int32_t mul_i32(int32_t a, int32_t b) { return (int32_t)((uint32_t)a * (uint32_t)b); }

static void set_threads(int threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ---------------------------------------------------------------------------
 * CSR vector-length hint.  loop_mapping.py:224-246 (_emit_hint, runtime case):
 *   k  = ceildivsi(rowptr[N], max(N, 1))
 *   VL = select chain over p = cap/2 .. 1 : (k <= p) ? p : previous
 * i.e. the smallest power of two p <= cap/2 with k <= p, else cap.  The
 * ceildivsi rounding follows runtime_header.py:75-80 / interp.py:492-495.
 * ------------------------------------------------------------------------- */
int64_t oracle_csr_vector_length(int64_t nrows, int64_t nnz, int64_t cap) {
  int64_t rows_floor = nrows > 1 ? nrows : 1;
  /* ceildivsi(a, b) = -((-a) // b) with floor division (interp.py:492-495) */
  int64_t na = -nnz, q = na / rows_floor;
  if ((na % rows_floor != 0) && ((na < 0) != (rows_floor < 0))) q -= 1;
  int64_t k = -q;
  int64_t acc = cap;
  for (int64_t p = cap / 2; p >= 1; p /= 2)
    if (k <= p) acc = p;
  return acc;
}

/* ---------------------------------------------------------------------------
 * sparse.spmv_csr — interp.py:798-812 (_h_spmv_csr):
 *   for i: acc = 0; for j in [rp[i], max(rp[i], rp[i+1])): acc += v[j]*x[ci[j]]
 *   y[i] = acc            (y overwritten, not accumulated)
 * Rows [row_begin, row_end) only (lets tests check sampled rows at full size).
 * ------------------------------------------------------------------------- */
void oracle_spmv_csr(int64_t row_begin, int64_t row_end,
                     const void* rowptr, int rp_bytes,
                     const void* colind, int ci_bytes,
                     const void* values, const void* x, void* y,
                     int dtype, int threads) {
  set_threads(threads);
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t i = row_begin; i < row_end; ++i) {
    int64_t b = ld_idx(rowptr, rp_bytes, i);
    int64_t e = ld_idx(rowptr, rp_bytes, i + 1);
    if (e < b) e = b;
    switch (dtype) {
      case OR_F64: {
        const double* v = (const double*)values; const double* xx = (const double*)x;
        double acc = 0.0;
        for (int64_t j = b; j < e; ++j) {
          double prod = v[j] * xx[ld_idx(colind, ci_bytes, j)];
          acc = acc + prod;
        }
        ((double*)y)[i] = acc;
        break;
      }
      case OR_F32: {
        const float* v = (const float*)values; const float* xx = (const float*)x;
        float acc = 0.0f;
        for (int64_t j = b; j < e; ++j) {
          float prod = v[j] * xx[ld_idx(colind, ci_bytes, j)];
          acc = acc + prod;
        }
        ((float*)y)[i] = acc;
        break;
      }
      case OR_I64: {
        const int64_t* v = (const int64_t*)values; const int64_t* xx = (const int64_t*)x;
        int64_t acc = 0;
        for (int64_t j = b; j < e; ++j)
          acc = add_i64(acc, mul_i64(v[j], xx[ld_idx(colind, ci_bytes, j)]));
        ((int64_t*)y)[i] = acc;
        break;
      }
      case OR_I32: {
        const int32_t* v = (const int32_t*)values; const int32_t* xx = (const int32_t*)x;
        int32_t acc = 0;
        for (int64_t j = b; j < e; ++j)
          acc = add_i32(acc, mul_i32(v[j], xx[ld_idx(colind, ci_bytes, j)]));
        ((int32_t*)y)[i] = acc;
        break;
      }
    }
  }
}

/* ---------------------------------------------------------------------------
 * CSR x dense SpMM.  The reference has no op for it; its loop-nest
 * form (oracle/ir/spmm.mlir, lowered by the reference pipeline to a
 * thread_parallel over N*K with the CSR hint) executes, per (i, c), the same
 * ascending sequential add-reduce as interp.py:798-812:
 *   Y[i, c] = sum_j v[j] * X[ci[j], c]
 * Row-major X (ldx) and Y (ldy), LayoutRight (runtime_header.py:39-41).
 * ------------------------------------------------------------------------- */
void oracle_spmm_csr(int64_t row_begin, int64_t row_end, int64_t k,
                     const void* rowptr, int rp_bytes,
                     const void* colind, int ci_bytes,
                     const void* values, const void* X, int64_t ldx,
                     void* Y, int64_t ldy, int dtype, int threads) {
  set_threads(threads);
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t i = row_begin; i < row_end; ++i) {
    int64_t b = ld_idx(rowptr, rp_bytes, i);
    int64_t e = ld_idx(rowptr, rp_bytes, i + 1);
    if (e < b) e = b;
    for (int64_t c = 0; c < k; ++c) {
      if (dtype == OR_F64) {
        const double* v = (const double*)values; const double* xx = (const double*)X;
        double acc = 0.0;
        for (int64_t j = b; j < e; ++j) {
          double prod = v[j] * xx[ld_idx(colind, ci_bytes, j) * ldx + c];
          acc = acc + prod;
        }
        ((double*)Y)[i * ldy + c] = acc;
      } else if (dtype == OR_F32) {
        const float* v = (const float*)values; const float* xx = (const float*)X;
        float acc = 0.0f;
        for (int64_t j = b; j < e; ++j) {
          float prod = v[j] * xx[ld_idx(colind, ci_bytes, j) * ldx + c];
          acc = acc + prod;
        }
        ((float*)Y)[i * ldy + c] = acc;
      } else if (dtype == OR_I64) {
        const int64_t* v = (const int64_t*)values; const int64_t* xx = (const int64_t*)X;
        int64_t acc = 0;
        for (int64_t j = b; j < e; ++j)
          acc = add_i64(acc, mul_i64(v[j], xx[ld_idx(colind, ci_bytes, j) * ldx + c]));
        ((int64_t*)Y)[i * ldy + c] = acc;
      } else {
        const int32_t* v = (const int32_t*)values; const int32_t* xx = (const int32_t*)X;
        int32_t acc = 0;
        for (int64_t j = b; j < e; ++j)
          acc = add_i32(acc, mul_i32(v[j], xx[ld_idx(colind, ci_bytes, j) * ldx + c]));
        ((int32_t*)Y)[i * ldy + c] = acc;
      }
    }
  }
}

/* ---------------------------------------------------------------------------
 * One dense dot product in the reference order: _matmul_impl / _matvec_impl
 * (interp.py:711-739): acc = 0; for k ascending: acc = round(acc + round(a*b)).
 * a has stride sa, b has stride sb (elements).
 * ------------------------------------------------------------------------- */
static void dot_seq(const void* a, int64_t sa, const void* b, int64_t sb, int64_t n,
                    void* out, int dtype) {
  switch (dtype) {
    case OR_F64: {
      const double* A = (const double*)a; const double* B = (const double*)b;
      double acc = 0.0;
      for (int64_t p = 0; p < n; ++p) { double prod = A[p * sa] * B[p * sb]; acc = acc + prod; }
      *(double*)out = acc; break;
    }
    case OR_F32: {
      const float* A = (const float*)a; const float* B = (const float*)b;
      float acc = 0.0f;
      for (int64_t p = 0; p < n; ++p) { float prod = A[p * sa] * B[p * sb]; acc = acc + prod; }
      *(float*)out = acc; break;
    }
    case OR_I64: {
      const int64_t* A = (const int64_t*)a; const int64_t* B = (const int64_t*)b;
      int64_t acc = 0;
      for (int64_t p = 0; p < n; ++p) acc = add_i64(acc, mul_i64(A[p * sa], B[p * sb]));
      *(int64_t*)out = acc; break;
    }
    case OR_I32: {
      const int32_t* A = (const int32_t*)a; const int32_t* B = (const int32_t*)b;
      int32_t acc = 0;
      for (int64_t p = 0; p < n; ++p) acc = add_i32(acc, mul_i32(A[p * sa], B[p * sb]));
      *(int32_t*)out = acc; break;
    }
  }
}

static size_t esize(int dtype) { return (dtype == OR_F64 || dtype == OR_I64) ? 8 : 4; }

/* linalg.matmul / kokkos.gemm — interp.py:711-722, 949-961.
 * C[i,j] = sum_k A[i,k] * B[k,j] for every (i, j) (row-major, leading dims). */
void oracle_matmul(int64_t m, int64_t n, int64_t k,
                   const void* A, int64_t lda, const void* B, int64_t ldb,
                   void* C, int64_t ldc, int dtype, int threads) {
  size_t es = esize(dtype);
  set_threads(threads);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j)
      dot_seq((const char*)A + (size_t)(i * lda) * es, 1,
              (const char*)B + (size_t)j * es, ldb, k,
              (char*)C + (size_t)(i * ldc + j) * es, dtype);
}

/* Selected entries of a matmul (full-size parity on sampled outputs). */
void oracle_matmul_entries(int64_t k, const void* A, int64_t lda, const void* B, int64_t ldb,
                           int64_t count, const int64_t* ii, const int64_t* jj, void* out,
                           int dtype, int threads) {
  size_t es = esize(dtype);
  set_threads(threads);
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < count; ++t)
    dot_seq((const char*)A + (size_t)(ii[t] * lda) * es, 1,
            (const char*)B + (size_t)jj[t] * es, ldb, k,
            (char*)out + (size_t)t * es, dtype);
}

/* linalg.matvec / kokkos.gemv — interp.py:729-739, 964-976. */
void oracle_matvec(int64_t m, int64_t n, const void* A, int64_t lda,
                   const void* x, void* y, int dtype, int threads) {
  size_t es = esize(dtype);
  set_threads(threads);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i)
    dot_seq((const char*)A + (size_t)(i * lda) * es, 1, x, 1, n,
            (char*)y + (size_t)i * es, dtype);
}

/* linalg.batch_matmul — interp.py:746-763.  Contiguous [b][m][k] x [b][k][n]. */
void oracle_batch_matmul(int64_t nb, int64_t m, int64_t n, int64_t k,
                         const void* A, const void* B, void* C, int dtype, int threads) {
  size_t es = esize(dtype);
  set_threads(threads);
#pragma omp parallel for schedule(static) collapse(2)
  for (int64_t t = 0; t < nb; ++t)
    for (int64_t i = 0; i < m; ++i)
      for (int64_t j = 0; j < n; ++j)
        dot_seq((const char*)A + (size_t)((t * m + i) * k) * es, 1,
                (const char*)B + (size_t)(t * k * n + j) * es, n, k,
                (char*)C + (size_t)((t * m + i) * n + j) * es, dtype);
}

/* ---------------------------------------------------------------------------
 * linalg.reduce on a rank-2 row-major array — interp.py:779-795 with combine
 * (interp.py:174-183) and combiner_identity (interp.py:186-195).
 * axis = 1: out[i] = fold_j src[i, j];  axis = 0: out[j] = fold_i src[i, j].
 * combiner: 0=add 1=mul 2=min 3=max (dialect.py:128-154 classify_combiner).
 * ------------------------------------------------------------------------- */
#define FOLD_BODY(T, ADD, MUL, IDENT_ADD, IDENT_MUL, IDENT_MIN, IDENT_MAX)          \
  {                                                                                \
    const T* S = (const T*)src; T* O = (T*)out;                                    \
    int64_t nout = axis == 1 ? rows : cols, nred = axis == 1 ? cols : rows;        \
    _Pragma("omp parallel for schedule(static)")                                   \
    for (int64_t o = 0; o < nout; ++o) {                                           \
      T acc = combiner == 0 ? IDENT_ADD : combiner == 1 ? IDENT_MUL                \
            : combiner == 2 ? IDENT_MIN : IDENT_MAX;                               \
      for (int64_t r = 0; r < nred; ++r) {                                         \
        T v = axis == 1 ? S[o * cols + r] : S[r * cols + o];                       \
        if (combiner == 0) acc = ADD(acc, v);                                      \
        else if (combiner == 1) acc = MUL(acc, v);                                 \
        else if (combiner == 2) acc = (acc <= v) ? acc : v;                        \
        else acc = (acc >= v) ? acc : v;                                           \
      }                                                                            \
      O[o] = acc;                                                                  \
    }                                                                              \
  }
static inline double fadd64(double a, double b) { return a + b; }
static inline double fmul64(double a, double b) { return a * b; }
static inline float fadd32(float a, float b) { return a + b; }
static inline float fmul32(float a, float b) { return a * b; }

void oracle_reduce2d(int64_t rows, int64_t cols, const void* src, void* out,
                     int axis, int combiner, int dtype, int threads) {
  set_threads(threads);
  switch (dtype) {
    case OR_F64: FOLD_BODY(double, fadd64, fmul64, 0.0, 1.0, INFINITY, -INFINITY) break;
    case OR_F32: FOLD_BODY(float, fadd32, fmul32, 0.0f, 1.0f, INFINITY, -INFINITY) break;
    case OR_I64: FOLD_BODY(int64_t, add_i64, mul_i64, 0, 1, INT64_MAX, INT64_MIN) break;
    case OR_I32: FOLD_BODY(int32_t, add_i32, mul_i32, 0, 1, INT32_MAX, INT32_MIN) break;
  }
}

/* GCN ReLU as the reference lowers linalg.elementwise{cmpf ogt; select}:
 * y = (x > 0) ? x : 0 (interp.py:520-545, 766-776).  NaN and -0.0 map to 0. */
void oracle_relu(int64_t n, const void* x, void* y, int dtype) {
  if (dtype == OR_F64) {
    for (int64_t i = 0; i < n; ++i) { double v = ((const double*)x)[i]; ((double*)y)[i] = v > 0.0 ? v : 0.0; }
  } else {
    for (int64_t i = 0; i < n; ++i) { float v = ((const float*)x)[i]; ((float*)y)[i] = v > 0.0f ? v : 0.0f; }
  }
}
