// Graph ingestion for the graph store (SPEC.md:121-129 load_graph, :160 External Interfaces):
//   edge file    text, one edge per line "src dest [edge_value]", whitespace separated,
//                base-10 non-negative ids; blank lines and lines starting with '#' or '%'
//                (SNAP / MatrixMarket comments) are skipped;
//   feature file text CSV (row v = features of vertex v; ',' and/or whitespace separated)
//                or raw binary: little-endian u64 rows, u64 cols, then row-major f64;
//   label file   one integer class per line.
// Files are memory-mapped and parsed in parallel (OpenMP) over newline-aligned slices;
// every error names the 1-based line.  Two-call pattern (scan sizes, then read into
// caller-owned buffers), no allocation crosses the ABI.
#include <fcntl.h>
#include <omp.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.h"

namespace {

struct MappedFile {
  const char* data = nullptr;
  size_t size = 0;
  int fd = -1;
  bool open(const char* path) {
    fd = ::open(path, O_RDONLY);
    if (fd < 0) return false;
    struct stat st;
    if (fstat(fd, &st) != 0) return false;
    size = (size_t)st.st_size;
    if (size == 0) return true;
    void* p = mmap(nullptr, size, PROT_READ, MAP_PRIVATE, fd, 0);
    if (p == MAP_FAILED) return false;
    madvise(p, size, MADV_SEQUENTIAL);
    data = static_cast<const char*>(p);
    return true;
  }
  ~MappedFile() {
    if (data) munmap(const_cast<char*>(data), size);
    if (fd >= 0) ::close(fd);
  }
};

// newline-aligned slices [b[k], b[k+1]) of the file, one per thread
std::vector<size_t> slices(const MappedFile& f, int n) {
  std::vector<size_t> b(n + 1, f.size);
  b[0] = 0;
  for (int k = 1; k < n; ++k) {
    size_t p = f.size * (size_t)k / (size_t)n;
    if (p < b[k - 1]) p = b[k - 1];
    while (p < f.size && p > 0 && f.data[p - 1] != '\n') ++p;
    b[k] = p;
  }
  return b;
}

inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\r'; }

// a line's fields, whitespace (and optionally comma) separated
struct Line {
  const char* p;
  const char* end;
};

inline bool skip_line(const Line& l) {
  const char* p = l.p;
  while (p < l.end && is_ws(*p)) ++p;
  return p == l.end || *p == '#' || *p == '%';
}

// parse a non-negative base-10 integer; returns false on junk / overflow
inline bool parse_uint(const char*& p, const char* end, uint64_t& v) {
  while (p < end && is_ws(*p)) ++p;
  if (p == end || *p < '0' || *p > '9') return false;
  uint64_t x = 0;
  while (p < end && *p >= '0' && *p <= '9') {
    x = x * 10 + (uint64_t)(*p - '0');
    if (x > (uint64_t)INT64_MAX) return false;
    ++p;
  }
  if (p < end && !is_ws(*p) && *p != ',') return false;
  v = x;
  return true;
}

inline bool parse_double(const char*& p, const char* end, double& v) {
  while (p < end && (is_ws(*p) || *p == ',')) ++p;
  if (p == end) return false;
  char buf[64];
  size_t n = 0;
  while (p + n < end && !is_ws(p[n]) && p[n] != ',' && n < sizeof(buf) - 1) {
    buf[n] = p[n];
    ++n;
  }
  buf[n] = 0;
  char* q = nullptr;
  errno = 0;
  v = strtod(buf, &q);
  if (q != buf + n || n == 0) return false;
  p += n;
  return true;
}

inline bool at_end(const char* p, const char* end) {
  while (p < end && (is_ws(*p) || *p == ',')) ++p;
  return p == end;
}

struct SliceStats {
  int64_t records = 0;   // data lines
  int64_t lines = 0;     // newline count (for global line numbers)
  int64_t bad_line = -1; // local 1-based line of the first error
  std::string why;
  int64_t max_id = -1;
  int ncols = -1;        // fields per line (edges: 2 or 3; matrices: cols)
};

template <typename Fn>
void for_lines(const MappedFile& f, size_t b, size_t e, Fn fn) {
  size_t p = b;
  int64_t ln = 0;
  while (p < e) {
    const char* s = f.data + p;
    const char* nl = static_cast<const char*>(memchr(s, '\n', e - p));
    const char* le = nl ? nl : f.data + e;
    ++ln;
    if (!fn(Line{s, le}, ln)) return;
    p = (size_t)(le - f.data) + 1;
  }
}

int64_t count_nl(const MappedFile& f, size_t b, size_t e) {
  int64_t n = 0;
  for (size_t p = b; p < e; ++p) n += f.data[p] == '\n';
  if (e > b && f.data[e - 1] != '\n') ++n;  // last line without newline
  return n;
}

// number of fields of an edge line (2 or 3), or -1 if malformed
int edge_fields(const Line& l, int64_t limit, uint64_t& s, uint64_t& d, double& val, std::string& why) {
  const char* p = l.p;
  if (!parse_uint(p, l.end, s) || !parse_uint(p, l.end, d)) {
    why = "expected 'src dest [edge_value]' with non-negative integer ids";
    return -1;
  }
  int n = 2;
  if (!at_end(p, l.end)) {
    if (!parse_double(p, l.end, val) || !at_end(p, l.end)) {
      why = "expected at most one numeric edge value after 'src dest'";
      return -1;
    }
    n = 3;
  }
  if (limit >= 0 && ((int64_t)s >= limit || (int64_t)d >= limit)) {
    why = "vertex id " + std::to_string(std::max(s, d)) + " out of range [0, " + std::to_string(limit) + ")";
    return -1;
  }
  if ((int64_t)std::max(s, d) > INT32_MAX - 1) {
    why = "vertex id exceeds the int32 id space";
    return -1;
  }
  return n;
}

int fail_line(const char* what, const char* path, int64_t line, const std::string& why) {
  SG_FAIL(SG_EFORMAT, "%s %s line %lld: %s", what, path, (long long)line, why.c_str());
}

// scan: per-slice records, errors (first in file order) and uniform field count
template <typename LineFn>
int scan_file(const char* what, const char* path, const MappedFile& f, std::vector<size_t>& b,
              std::vector<SliceStats>& st, LineFn fn) {
  const int T = (int)b.size() - 1;
#pragma omp parallel for schedule(static, 1) num_threads(T)
  for (int k = 0; k < T; ++k) {
    SliceStats& s = st[k];
    s.lines = count_nl(f, b[k], b[k + 1]);
    for_lines(f, b[k], b[k + 1], [&](const Line& l, int64_t ln) { return fn(l, ln, s); });
  }
  int64_t line0 = 0;
  int ncols = -1;
  for (int k = 0; k < T; ++k) {
    if (st[k].bad_line >= 0) return fail_line(what, path, line0 + st[k].bad_line, st[k].why);
    line0 += st[k].lines;
  }
  // consistent field count across slices
  line0 = 0;
  for (int k = 0; k < T; ++k) {
    if (st[k].ncols >= 0) {
      if (ncols >= 0 && st[k].ncols != ncols)
        SG_FAIL(SG_EFORMAT, "%s %s: rows have different field counts (%d vs %d)", what, path, ncols,
                st[k].ncols);
      ncols = st[k].ncols;
    }
  }
  return SG_OK;
}

int nthreads_for(size_t bytes) {
  const int t = std::max(1, omp_get_max_threads());
  return (int)std::max<size_t>(1, std::min<size_t>((size_t)t, bytes / (1 << 20) + 1));
}

}  // namespace

extern "C" {

int sg_host_scan_edges(const char* path, int64_t vertex_limit, int64_t* n_edges, int64_t* max_id,
                       int* has_value) {
  SG_REQUIRE(path && n_edges && max_id && has_value, SG_EINVAL, "scan_edges: null argument");
  MappedFile f;
  if (!f.open(path)) SG_FAIL(SG_EFORMAT, "cannot open edge file %s: %s", path, strerror(errno));
  auto b = slices(f, nthreads_for(f.size));
  std::vector<SliceStats> st(b.size() - 1);
  int rc = scan_file("edge file", path, f, b, st, [&](const Line& l, int64_t ln, SliceStats& s) {
    if (skip_line(l)) return true;
    uint64_t u, v;
    double val;
    int n = edge_fields(l, vertex_limit, u, v, val, s.why);
    if (n < 0 || (s.ncols >= 0 && n != s.ncols)) {
      if (n >= 0) s.why = "edge value present on some lines but not others";
      s.bad_line = ln;
      return false;
    }
    s.ncols = n;
    s.records++;
    s.max_id = std::max<int64_t>(s.max_id, (int64_t)std::max(u, v));
    return true;
  });
  if (rc != SG_OK) return rc;
  int64_t E = 0, m = -1;
  int nc = -1;
  for (auto& s : st) {
    E += s.records;
    m = std::max(m, s.max_id);
    if (s.ncols >= 0) nc = s.ncols;
  }
  *n_edges = E;
  *max_id = m;
  *has_value = nc == 3;
  return SG_OK;
}

int sg_host_read_edges(const char* path, int64_t n_edges, int32_t* src, int32_t* dst, double* value) {
  SG_REQUIRE(path && (n_edges == 0 || (src && dst)), SG_EINVAL, "read_edges: null argument");
  MappedFile f;
  if (!f.open(path)) SG_FAIL(SG_EFORMAT, "cannot open edge file %s: %s", path, strerror(errno));
  auto b = slices(f, nthreads_for(f.size));
  const int T = (int)b.size() - 1;
  std::vector<int64_t> cnt(T + 1, 0);
#pragma omp parallel for schedule(static, 1) num_threads(T)
  for (int k = 0; k < T; ++k) {
    int64_t c = 0;
    for_lines(f, b[k], b[k + 1], [&](const Line& l, int64_t) {
      c += !skip_line(l);
      return true;
    });
    cnt[k + 1] = c;
  }
  for (int k = 0; k < T; ++k) cnt[k + 1] += cnt[k];
  SG_REQUIRE(cnt[T] == n_edges, SG_EFORMAT, "edge file %s changed between scan and read", path);
#pragma omp parallel for schedule(static, 1) num_threads(T)
  for (int k = 0; k < T; ++k) {
    int64_t o = cnt[k];
    std::string why;
    for_lines(f, b[k], b[k + 1], [&](const Line& l, int64_t) {
      if (skip_line(l)) return true;
      uint64_t u = 0, v = 0;
      double val = 0.0;
      edge_fields(l, -1, u, v, val, why);
      src[o] = (int32_t)u;
      dst[o] = (int32_t)v;
      if (value) value[o] = val;
      ++o;
      return true;
    });
  }
  return SG_OK;
}

int sg_host_scan_matrix_text(const char* path, int64_t* rows, int64_t* cols) {
  SG_REQUIRE(path && rows && cols, SG_EINVAL, "scan_matrix_text: null argument");
  MappedFile f;
  if (!f.open(path)) SG_FAIL(SG_EFORMAT, "cannot open feature file %s: %s", path, strerror(errno));
  auto b = slices(f, nthreads_for(f.size));
  std::vector<SliceStats> st(b.size() - 1);
  int rc = scan_file("feature file", path, f, b, st, [&](const Line& l, int64_t ln, SliceStats& s) {
    if (skip_line(l)) return true;
    const char* p = l.p;
    int n = 0;
    double v;
    while (!at_end(p, l.end)) {
      if (!parse_double(p, l.end, v)) {
        s.why = "expected numeric fields separated by ',' or whitespace";
        s.bad_line = ln;
        return false;
      }
      ++n;
    }
    if (s.ncols >= 0 && n != s.ncols) {
      s.why = "row has " + std::to_string(n) + " fields, previous rows " + std::to_string(s.ncols);
      s.bad_line = ln;
      return false;
    }
    s.ncols = n;
    s.records++;
    return true;
  });
  if (rc != SG_OK) return rc;
  int64_t R = 0;
  int C = 0;
  for (auto& s : st) {
    R += s.records;
    if (s.ncols >= 0) C = s.ncols;
  }
  *rows = R;
  *cols = C;
  return SG_OK;
}

int sg_host_read_matrix_text(const char* path, int64_t rows, int64_t cols, double* out) {
  SG_REQUIRE(path && (rows * cols == 0 || out), SG_EINVAL, "read_matrix_text: null argument");
  MappedFile f;
  if (!f.open(path)) SG_FAIL(SG_EFORMAT, "cannot open feature file %s: %s", path, strerror(errno));
  auto b = slices(f, nthreads_for(f.size));
  const int T = (int)b.size() - 1;
  std::vector<int64_t> cnt(T + 1, 0);
#pragma omp parallel for schedule(static, 1) num_threads(T)
  for (int k = 0; k < T; ++k) {
    int64_t c = 0;
    for_lines(f, b[k], b[k + 1], [&](const Line& l, int64_t) {
      c += !skip_line(l);
      return true;
    });
    cnt[k + 1] = c;
  }
  for (int k = 0; k < T; ++k) cnt[k + 1] += cnt[k];
  SG_REQUIRE(cnt[T] == rows, SG_EFORMAT, "feature file %s changed between scan and read", path);
#pragma omp parallel for schedule(static, 1) num_threads(T)
  for (int k = 0; k < T; ++k) {
    int64_t r = cnt[k];
    for_lines(f, b[k], b[k + 1], [&](const Line& l, int64_t) {
      if (skip_line(l)) return true;
      const char* p = l.p;
      for (int64_t c = 0; c < cols; ++c) {
        double v = 0.0;
        parse_double(p, l.end, v);
        out[r * cols + c] = v;
      }
      ++r;
      return true;
    });
  }
  return SG_OK;
}

int sg_host_read_matrix_bin_header(const char* path, int64_t* rows, int64_t* cols) {
  SG_REQUIRE(path && rows && cols, SG_EINVAL, "read_matrix_bin_header: null argument");
  FILE* fp = fopen(path, "rb");
  if (!fp) SG_FAIL(SG_EFORMAT, "cannot open feature file %s: %s", path, strerror(errno));
  uint64_t h[2] = {0, 0};
  const size_t got = fread(h, 8, 2, fp);
  fseek(fp, 0, SEEK_END);
  const long size = ftell(fp);
  fclose(fp);
  SG_REQUIRE(got == 2, SG_EFORMAT, "feature file %s: missing u64 rows/cols header", path);
  SG_REQUIRE(h[0] < (1ull << 40) && h[1] < (1ull << 32), SG_EFORMAT, "feature file %s: bad header %llu x %llu",
             path, (unsigned long long)h[0], (unsigned long long)h[1]);
  const uint64_t need = 16 + h[0] * h[1] * 8;
  SG_REQUIRE((uint64_t)size == need, SG_EFORMAT,
             "feature file %s: %ld bytes, header %llu x %llu f64 needs %llu", path, size,
             (unsigned long long)h[0], (unsigned long long)h[1], (unsigned long long)need);
  *rows = (int64_t)h[0];
  *cols = (int64_t)h[1];
  return SG_OK;
}

int sg_host_read_matrix_bin(const char* path, int64_t rows, int64_t cols, double* out) {
  int64_t r = 0, c = 0;
  int rc = sg_host_read_matrix_bin_header(path, &r, &c);
  if (rc != SG_OK) return rc;
  SG_REQUIRE(r == rows && c == cols, SG_EFORMAT, "feature file %s: header %lld x %lld, expected %lld x %lld",
             path, (long long)r, (long long)c, (long long)rows, (long long)cols);
  MappedFile f;
  if (!f.open(path)) SG_FAIL(SG_EFORMAT, "cannot open feature file %s: %s", path, strerror(errno));
  const size_t n = (size_t)rows * (size_t)cols;
  const int T = nthreads_for(n * 8);
#pragma omp parallel for num_threads(T)
  for (int k = 0; k < T; ++k) {
    const size_t a = n * (size_t)k / (size_t)T, e = n * (size_t)(k + 1) / (size_t)T;
    if (e > a) memcpy(out + a, f.data + 16 + a * 8, (e - a) * 8);
  }
  return SG_OK;
}

int sg_host_write_matrix_bin(const char* path, int64_t rows, int64_t cols, const double* data) {
  SG_REQUIRE(path && rows >= 0 && cols >= 0 && (rows * cols == 0 || data), SG_EINVAL,
             "write_matrix_bin: bad argument");
  FILE* fp = fopen(path, "wb");
  if (!fp) SG_FAIL(SG_EFORMAT, "cannot create %s: %s", path, strerror(errno));
  const uint64_t h[2] = {(uint64_t)rows, (uint64_t)cols};
  bool ok = fwrite(h, 8, 2, fp) == 2;
  if (rows * cols) ok = ok && fwrite(data, 8, (size_t)(rows * cols), fp) == (size_t)(rows * cols);
  ok = (fclose(fp) == 0) && ok;
  SG_REQUIRE(ok, SG_EFORMAT, "short write to %s", path);
  return SG_OK;
}

int sg_host_scan_labels(const char* path, int64_t* n) {
  SG_REQUIRE(path && n, SG_EINVAL, "scan_labels: null argument");
  MappedFile f;
  if (!f.open(path)) SG_FAIL(SG_EFORMAT, "cannot open label file %s: %s", path, strerror(errno));
  auto b = slices(f, nthreads_for(f.size));
  std::vector<SliceStats> st(b.size() - 1);
  int rc = scan_file("label file", path, f, b, st, [&](const Line& l, int64_t ln, SliceStats& s) {
    if (skip_line(l)) return true;
    const char* p = l.p;
    uint64_t v;
    if (!parse_uint(p, l.end, v) || !at_end(p, l.end)) {
      s.why = "expected one non-negative integer class";
      s.bad_line = ln;
      return false;
    }
    s.records++;
    return true;
  });
  if (rc != SG_OK) return rc;
  int64_t N = 0;
  for (auto& s : st) N += s.records;
  *n = N;
  return SG_OK;
}

int sg_host_read_labels(const char* path, int64_t n, int64_t* out) {
  SG_REQUIRE(path && (n == 0 || out), SG_EINVAL, "read_labels: null argument");
  MappedFile f;
  if (!f.open(path)) SG_FAIL(SG_EFORMAT, "cannot open label file %s: %s", path, strerror(errno));
  int64_t i = 0;
  for_lines(f, 0, f.size, [&](const Line& l, int64_t) {
    if (skip_line(l)) return true;
    if (i >= n) return false;
    const char* p = l.p;
    uint64_t v = 0;
    parse_uint(p, l.end, v);
    out[i++] = (int64_t)v;
    return true;
  });
  SG_REQUIRE(i == n, SG_EFORMAT, "label file %s changed between scan and read", path);
  return SG_OK;
}

// 64-bit content hash (order-sensitive) of a byte buffer, parallel over 1 MiB blocks:
// keys the on-disk partition cache.
uint64_t sg_host_hash64(const void* data, int64_t nbytes, uint64_t seed) {
  const unsigned char* p = static_cast<const unsigned char*>(data);
  const int64_t B = 1 << 20;
  const int64_t nb = (nbytes + B - 1) / B;
  std::vector<uint64_t> hb((size_t)std::max<int64_t>(nb, 1), 0);
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < nb; ++k) {
    const int64_t a = k * B, e = std::min(nbytes, a + B);
    uint64_t h = 0x9E3779B97F4A7C15ull ^ (uint64_t)k;
    int64_t i = a;
    for (; i + 8 <= e; i += 8) {
      uint64_t w;
      memcpy(&w, p + i, 8);
      h ^= w;
      h *= 0xBF58476D1CE4E5B9ull;
      h ^= h >> 31;
    }
    for (; i < e; ++i) {
      h ^= p[i];
      h *= 0x94D049BB133111EBull;
    }
    hb[(size_t)k] = h;
  }
  uint64_t h = seed ^ (uint64_t)nbytes;
  for (int64_t k = 0; k < nb; ++k) {
    h ^= hb[(size_t)k] + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
  }
  return h;
}

}  // extern "C"
