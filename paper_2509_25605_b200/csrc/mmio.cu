// mmio.cu — Matrix Market (coordinate) reader straight into CSR, host side.
//
// the paper's SpMV study runs SuiteSparse matrices
// (StocF-1465, PFlow_742, audikw_1, Elasticity3D), which ship
// as Matrix Market files; the reference has no reader (its inputs are the
// `shape: / data: / file:` args format, tensors.py:25-104).  This reader maps
// the file, parses the entry lines in parallel (one std::thread per chunk of
// lines), expands symmetric / skew-symmetric / hermitian storage, and builds a
// row-sorted CSR (int64 rowptr, int32 or int64 colind, f64 values) in two
// passes (row counts -> prefix sums -> scatter -> per-row column sort), the
// layout the B200 kernels stream.  Host code only: no device is touched.
#include "common.cuh"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cctype>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

namespace lapis_b200 {
namespace {

enum Field { REAL = 0, INTEGER = 1, PATTERN = 2, COMPLEX = 3 };
enum Sym { GENERAL = 0, SYMMETRIC = 1, SKEW = 2, HERMITIAN = 3 };

struct Mapped {
  const char* p = nullptr;
  size_t n = 0;
  int fd = -1;
  ~Mapped() {
    if (p) munmap(const_cast<char*>(p), n);
    if (fd >= 0) close(fd);
  }
};

struct Header {
  int field = REAL, sym = GENERAL;
  int64_t nrows = 0, ncols = 0, nentries = 0;
  size_t body = 0;  // offset of the first entry line
};

std::string lower(std::string s) {
  for (auto& c : s) c = (char)std::tolower((unsigned char)c);
  return s;
}

int map_file(const char* path, Mapped& m) {
  m.fd = open(path, O_RDONLY);
  if (m.fd < 0) return fail(LAPIS_B200_ERR_ARG, std::string("matrix market: cannot open ") + path);
  struct stat st;
  if (fstat(m.fd, &st) != 0 || st.st_size <= 0)
    return fail(LAPIS_B200_ERR_ARG, std::string("matrix market: empty file ") + path);
  m.n = (size_t)st.st_size;
  void* p = mmap(nullptr, m.n, PROT_READ, MAP_PRIVATE, m.fd, 0);
  if (p == MAP_FAILED) return fail(LAPIS_B200_ERR_ARG, "matrix market: mmap failed");
  m.p = static_cast<const char*>(p);
  return LAPIS_B200_OK;
}

int parse_header(const Mapped& m, Header& h) {
  size_t i = 0;
  auto line_end = [&](size_t s) {
    const void* e = memchr(m.p + s, '\n', m.n - s);
    return e ? (size_t)(static_cast<const char*>(e) - m.p) : m.n;
  };
  size_t e = line_end(0);
  std::string banner = lower(std::string(m.p, e));
  if (banner.rfind("%%matrixmarket", 0) != 0)
    return fail(LAPIS_B200_ERR_ARG, "matrix market: missing %%MatrixMarket banner");
  if (banner.find("coordinate") == std::string::npos)
    return fail(LAPIS_B200_ERR_UNSUPPORTED, "matrix market: only coordinate (sparse) matrices");
  if (banner.find("complex") != std::string::npos)
    return fail(LAPIS_B200_ERR_UNSUPPORTED, "matrix market: complex values are not supported");
  h.field = banner.find("pattern") != std::string::npos ? PATTERN
            : banner.find("integer") != std::string::npos ? INTEGER : REAL;
  h.sym = banner.find("skew-symmetric") != std::string::npos ? SKEW
          : banner.find("symmetric") != std::string::npos ? SYMMETRIC
          : banner.find("hermitian") != std::string::npos ? HERMITIAN : GENERAL;
  i = e + 1;
  while (i < m.n) {  // comments and blank lines
    e = line_end(i);
    size_t k = i;
    while (k < e && (m.p[k] == ' ' || m.p[k] == '\t' || m.p[k] == '\r')) ++k;
    if (k < e && m.p[k] != '%') break;
    i = e + 1;
  }
  if (i >= m.n) return fail(LAPIS_B200_ERR_ARG, "matrix market: missing size line");
  e = line_end(i);
  std::string size_line(m.p + i, e - i);
  long long r = 0, c = 0, z = 0;
  if (sscanf(size_line.c_str(), "%lld %lld %lld", &r, &c, &z) != 3 || r < 0 || c < 0 || z < 0)
    return fail(LAPIS_B200_ERR_ARG, "matrix market: bad size line");
  h.nrows = r;
  h.ncols = c;
  h.nentries = z;
  h.body = e + 1;
  return LAPIS_B200_OK;
}

struct Entry {
  int64_t r, c;
  double v;
};

inline const char* skip_ws(const char* p, const char* end) {
  while (p < end && (*p == ' ' || *p == '\t' || *p == '\r')) ++p;
  return p;
}

// parse the entry lines of [begin, end) (line-aligned) into `out`
int parse_chunk(const char* begin, const char* end, int field, std::vector<Entry>& out,
                std::string& err) {
  const char* p = begin;
  while (p < end) {
    const char* nl = static_cast<const char*>(memchr(p, '\n', end - p));
    const char* le = nl ? nl : end;
    const char* q = skip_ws(p, le);
    if (q < le && *q != '%') {
      char* tail = nullptr;
      const long long r = strtoll(q, &tail, 10);
      q = tail;
      const long long c = strtoll(q, &tail, 10);
      if (tail == q) { err = "matrix market: bad entry line"; return LAPIS_B200_ERR_ARG; }
      q = tail;
      double v = 1.0;
      if (field != PATTERN) {
        v = strtod(q, &tail);
        if (tail == q) { err = "matrix market: entry without a value"; return LAPIS_B200_ERR_ARG; }
      }
      out.push_back({r - 1, c - 1, v});
    }
    p = le + 1;
  }
  return LAPIS_B200_OK;
}

struct Parsed {
  Header h;
  std::vector<std::vector<Entry>> chunks;
};

int parse_all(const char* path, Parsed& out) {
  Mapped m;
  LB_TRY(map_file(path, m));
  LB_TRY(parse_header(m, out.h));
  const char* body = m.p + out.h.body;
  const char* end = m.p + m.n;
  const size_t len = body < end ? (size_t)(end - body) : 0;
  unsigned nt = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
  if (len < (1u << 20)) nt = 1;
  std::vector<const char*> cuts(nt + 1, end);
  cuts[0] = body;
  for (unsigned t = 1; t < nt; ++t) {  // line-aligned split points
    const char* c = body + len * t / nt;
    if (c < cuts[t - 1]) c = cuts[t - 1];
    const char* nl = static_cast<const char*>(memchr(c, '\n', end - c));
    cuts[t] = nl ? nl + 1 : end;
  }
  out.chunks.assign(nt, {});
  std::vector<int> rc(nt, LAPIS_B200_OK);
  std::vector<std::string> err(nt);
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      out.chunks[t].reserve((size_t)(out.h.nentries / nt + 16));
      rc[t] = parse_chunk(cuts[t], cuts[t + 1], out.h.field, out.chunks[t], err[t]);
    });
  for (auto& x : th) x.join();
  size_t total = 0;
  for (unsigned t = 0; t < nt; ++t) {
    if (rc[t] != LAPIS_B200_OK) return fail(rc[t], err[t]);
    total += out.chunks[t].size();
  }
  if ((int64_t)total != out.h.nentries)
    return fail(LAPIS_B200_ERR_ARG, "matrix market: entry count differs from the size line");
  for (auto& ch : out.chunks)
    for (const Entry& x : ch)
      if (x.r < 0 || x.r >= out.h.nrows || x.c < 0 || x.c >= out.h.ncols)
        return fail(LAPIS_B200_ERR_ARG, "matrix market: entry index out of range");
  return LAPIS_B200_OK;
}

inline bool mirrored(const Header& h, const Entry& x) { return h.sym != GENERAL && x.r != x.c; }

}  // namespace
}  // namespace lapis_b200

using namespace lapis_b200;

extern "C" {

// Size of the CSR the file expands to: out4 = {nrows, ncols, nnz (symmetric
// storage expanded), flags: bit0 pattern, bit1 integer, bits 2-3 symmetry}.
int lapis_b200_mm_info(const char* path, int64_t* out4) {
  if (!path || !out4) return fail(LAPIS_B200_ERR_ARG, "mm_info: null argument");
  Parsed ps;
  LB_TRY(parse_all(path, ps));
  int64_t nnz = 0;
  for (auto& ch : ps.chunks)
    for (const Entry& x : ch) nnz += mirrored(ps.h, x) ? 2 : 1;
  out4[0] = ps.h.nrows;
  out4[1] = ps.h.ncols;
  out4[2] = nnz;
  out4[3] = (ps.h.field == PATTERN ? 1 : 0) | (ps.h.field == INTEGER ? 2 : 0) | (ps.h.sym << 2);
  return LAPIS_B200_OK;
}

// Fill host CSR arrays sized by lapis_b200_mm_info: rowptr [nrows + 1] int64,
// colind [nnz] (colind_bytes 4 or 8), values [nnz] f64 (may be NULL for a
// structure-only read).  Rows sorted by column; duplicate entries are kept in
// file order (Matrix Market files do not repeat coordinates).
int lapis_b200_mm_read_csr(const char* path, int64_t* rowptr, void* colind, int colind_bytes,
                           double* values) {
  LB_RANGE("lapis_b200_mm_read_csr");
  if (!path || !rowptr || !colind) return fail(LAPIS_B200_ERR_ARG, "mm_read_csr: null argument");
  if (colind_bytes != 4 && colind_bytes != 8)
    return fail(LAPIS_B200_ERR_ARG, "mm_read_csr: colind_bytes must be 4 or 8");
  Parsed ps;
  LB_TRY(parse_all(path, ps));
  const Header& h = ps.h;
  if (colind_bytes == 4 && h.ncols > 0x7fffffffLL)
    return fail(LAPIS_B200_ERR_ARG, "mm_read_csr: columns exceed int32");
  std::vector<int64_t> cnt((size_t)h.nrows + 1, 0);
  for (auto& ch : ps.chunks)
    for (const Entry& x : ch) {
      ++cnt[(size_t)x.r + 1];
      if (mirrored(h, x)) ++cnt[(size_t)x.c + 1];
    }
  for (int64_t r = 0; r < h.nrows; ++r) cnt[(size_t)r + 1] += cnt[(size_t)r];
  std::memcpy(rowptr, cnt.data(), cnt.size() * sizeof(int64_t));
  const int64_t nnz = cnt[(size_t)h.nrows];
  std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
  std::vector<int64_t> col((size_t)nnz);
  std::vector<double> val((size_t)nnz);
  const double mirror_sign = h.sym == SKEW ? -1.0 : 1.0;
  for (auto& ch : ps.chunks)
    for (const Entry& x : ch) {
      int64_t k = pos[(size_t)x.r]++;
      col[(size_t)k] = x.c;
      val[(size_t)k] = x.v;
      if (mirrored(h, x)) {
        k = pos[(size_t)x.c]++;
        col[(size_t)k] = x.r;
        val[(size_t)k] = mirror_sign * x.v;
      }
    }
  // per-row column sort (stable: equal columns keep file order), parallel over rows
  const unsigned nt = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      std::vector<int64_t> idx;
      std::vector<int64_t> c2;
      std::vector<double> v2;
      for (int64_t r = t; r < h.nrows; r += nt) {
        const int64_t b = cnt[(size_t)r], e = cnt[(size_t)r + 1];
        if (e - b < 2) continue;
        bool sorted = true;
        for (int64_t k = b + 1; k < e && sorted; ++k) sorted = col[(size_t)k - 1] <= col[(size_t)k];
        if (sorted) continue;
        idx.resize((size_t)(e - b));
        std::iota(idx.begin(), idx.end(), b);
        std::stable_sort(idx.begin(), idx.end(),
                         [&](int64_t a, int64_t z) { return col[(size_t)a] < col[(size_t)z]; });
        c2.resize(idx.size());
        v2.resize(idx.size());
        for (size_t q = 0; q < idx.size(); ++q) {
          c2[q] = col[(size_t)idx[q]];
          v2[q] = val[(size_t)idx[q]];
        }
        std::copy(c2.begin(), c2.end(), col.begin() + b);
        std::copy(v2.begin(), v2.end(), val.begin() + b);
      }
    });
  for (auto& x : th) x.join();
  if (colind_bytes == 8) {
    std::memcpy(colind, col.data(), (size_t)nnz * 8);
  } else {
    int32_t* c32 = static_cast<int32_t*>(colind);
    for (int64_t k = 0; k < nnz; ++k) c32[k] = (int32_t)col[(size_t)k];
  }
  if (values) std::memcpy(values, val.data(), (size_t)nnz * sizeof(double));
  return LAPIS_B200_OK;
}

}  // extern "C"
