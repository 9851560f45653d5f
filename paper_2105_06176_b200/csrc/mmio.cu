// mmio.cu -- Matrix Market ingestion.
//
// Restates the reference parser sparse.py:195-326 (parse_matrix_market /
// load_matrix_market) with the same accepted subset (`matrix coordinate
// real general|symmetric`), the same checks in the same order and the same
// 1-based line numbers in its errors, but built for 10^8-nonzero files:
//
//  * host: the document is split at line boundaries into one chunk per
//    thread; every thread tokenises its chunk (std::from_chars, correctly
//    rounded like Python's float()) into a local COO list; errors are
//    ordered by document position afterwards, so the first error the
//    reference would raise is the one reported;
//  * device: COO -> CSR with a stable radix sort of (row, col) keys (CUB),
//    duplicates summed in the reference's np.add.reduceat order, row
//    offsets by count + scan.
//    The resulting CSR is left in HBM (the solve does not upload it again)
//    and copied back for the host CsrMatrix the reference API returns.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/pipecg_b200.h"
#include "internal.h"

struct pcg_mm {
  int64_t n_rows = 0, n_cols = 0, n_coo = 0;
  std::vector<int64_t> key;  // row * n_cols + col, document order (mirrored entries appended)
  std::vector<double> val;
};

namespace pcg {
namespace {

// Python str.split()/strip() whitespace (ASCII part)
inline bool is_ws(char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f' ||
         (c >= 0x1c && c <= 0x1f);
}

struct Line {
  const char* b;
  const char* e;
};

// next line starting at p (universal newlines: \n, \r\n, \r), or false at end
inline bool next_line(const char*& p, const char* end, bool universal, Line* out) {
  if (p >= end) return false;
  const char* q = p;
  while (q < end && *q != '\n' && !(universal && *q == '\r')) ++q;
  out->b = p;
  out->e = q;
  if (q < end) {
    if (*q == '\r' && q + 1 < end && q[1] == '\n') ++q;
    ++q;
  }
  p = q;
  return true;
}

inline void strip(Line* l) {
  while (l->b < l->e && is_ws(*l->b)) ++l->b;
  while (l->e > l->b && is_ws(l->e[-1])) --l->e;
}

// split on whitespace into at most `cap` tokens; returns the token count
// (counting beyond cap)
inline int split(Line l, Line* tok, int cap) {
  int n = 0;
  const char* p = l.b;
  while (p < l.e) {
    while (p < l.e && is_ws(*p)) ++p;
    if (p >= l.e) break;
    const char* s = p;
    while (p < l.e && !is_ws(*p)) ++p;
    if (n < cap) tok[n] = Line{s, p};
    ++n;
  }
  return n;
}

inline std::string str(Line l) { return std::string(l.b, l.e); }

// Python repr of an ASCII token ('...' unless it contains a quote)
std::string py_repr(const std::string& s) {
  const bool sq = s.find('\'') != std::string::npos, dq = s.find('"') != std::string::npos;
  const char q = sq && !dq ? '"' : '\'';
  std::string out(1, q);
  for (char c : s) {
    if (c == '\\') out += "\\\\";
    else if (c == q) out += std::string("\\") + q;
    else if (c == '\t') out += "\\t";
    else if ((unsigned char)c < 0x20 || (unsigned char)c >= 0x7f) {
      char buf[8];
      snprintf(buf, sizeof buf, "\\x%02x", (unsigned char)c);
      out += buf;
    } else out += c;
  }
  return out + q;
}

// Python int(token): [+-] digit (['_'] digit)*.  *big = true if it does not
// fit int64 (value then irrelevant; `norm` holds the decimal form).
bool py_int(Line t, int64_t* v, bool* big, std::string* norm) {
  // fast path: plain digits that fit
  if (t.e - t.b <= 18 && t.e > t.b) {
    int64_t x = 0;
    const char* q = t.b;
    for (; q < t.e && *q >= '0' && *q <= '9'; ++q) x = x * 10 + (*q - '0');
    if (q == t.e) {
      *v = x;
      *big = false;
      if (norm) *norm = std::to_string(x);
      return true;
    }
  }
  const char* p = t.b;
  bool neg = false;
  if (p < t.e && (*p == '+' || *p == '-')) neg = *p++ == '-';
  if (p >= t.e) return false;
  std::string digits;
  bool prev_digit = false;
  for (; p < t.e; ++p) {
    if (*p >= '0' && *p <= '9') {
      digits += *p;
      prev_digit = true;
    } else if (*p == '_' && prev_digit && p + 1 < t.e && p[1] >= '0' && p[1] <= '9') {
      prev_digit = false;
    } else {
      return false;
    }
  }
  size_t nz = digits.find_first_not_of('0');
  digits = nz == std::string::npos ? "0" : digits.substr(nz);
  if (norm) *norm = (neg && digits != "0" ? "-" : "") + digits;
  *big = digits.size() > 18;
  if (!*big) {
    int64_t x = 0;
    for (char c : digits) x = x * 10 + (c - '0');
    *v = neg ? -x : x;
  }
  return true;
}

// Python float(token) grammar, then correctly rounded conversion
bool py_float_once(const std::string& s, double* v) {
  const char* p = s.data();
  const char* e = p + s.size();
  bool neg = false;
  if (p < e && (*p == '+' || *p == '-')) neg = *p++ == '-';
  std::string body(p, e);
  std::string low;
  for (char c : body) low += (char)tolower((unsigned char)c);
  if (low == "inf" || low == "infinity") {
    *v = neg ? -HUGE_VAL : HUGE_VAL;
    return true;
  }
  if (low == "nan") {
    *v = neg ? -NAN : NAN;
    return true;
  }
  // digitpart ('.' digitpart?)? | '.' digitpart, exponent? ; '_' only between digits
  std::string clean;
  size_t i = 0, n = body.size();
  auto digitpart = [&](bool required) {
    size_t start = i;
    bool prev = false;
    while (i < n) {
      const char c = body[i];
      if (c >= '0' && c <= '9') {
        clean += c;
        prev = true;
        ++i;
      } else if (c == '_' && prev && i + 1 < n && body[i + 1] >= '0' && body[i + 1] <= '9') {
        prev = false;
        ++i;
      } else break;
    }
    return !required || i > start;
  };
  const bool has_int = digitpart(false) && !clean.empty();
  bool has_frac = false;
  if (i < n && body[i] == '.') {
    clean += '.';
    ++i;
    const size_t before = clean.size();
    digitpart(false);
    has_frac = clean.size() > before;
  }
  if (!has_int && !has_frac) return false;
  if (i < n && (body[i] == 'e' || body[i] == 'E')) {
    clean += 'e';
    ++i;
    if (i < n && (body[i] == '+' || body[i] == '-')) clean += body[i++];
    const size_t before = clean.size();
    digitpart(false);
    if (clean.size() == before) return false;
  }
  if (i != n) return false;
  double x = 0.0;
  auto r = std::from_chars(clean.data(), clean.data() + clean.size(), x);
  if (r.ec == std::errc::result_out_of_range) {
    // overflow / subnormal / underflow: strtod rounds these like Python's
    // float() (inf, the correctly rounded subnormal, or 0)
    x = strtod(clean.c_str(), nullptr);
  } else if (r.ec != std::errc() || r.ptr != clean.data() + clean.size()) {
    return false;
  }
  *v = neg ? -x : x;
  return true;
}

// _parse_float (sparse.py:183-192): Fortran 'd' exponents retried
bool py_float(Line t, double* v) {
  // fast path: [-]digits[.digits][e[+-]digits] is parsed identically by
  // from_chars and Python's float()
  {
    bool plain = t.e > t.b;
    for (const char* q = t.b; q < t.e && plain; ++q) {
      const char c = *q;
      plain = (c >= '0' && c <= '9') || c == '.' || c == 'e' || c == 'E' || c == '-' || c == '+';
    }
    if (plain && *t.b != '+') {
      double x = 0.0;
      auto r = std::from_chars(t.b, t.e, x);
      if (r.ec == std::errc() && r.ptr == t.e) {
        *v = x;
        return true;
      }
    }
  }
  std::string s = str(t);
  if (py_float_once(s, v)) return true;
  for (char& c : s) {
    if (c == 'd') c = 'e';
    else if (c == 'D') c = 'E';
  }
  return py_float_once(s, v);
}

struct Chunk {
  const char* b;
  const char* e;
  int64_t n_lines = 0;          // lines in the chunk
  std::vector<int32_t> row, col;  // 0-based
  std::vector<double> val;
  int64_t n_off = 0;            // off-diagonal entries (mirrored if symmetric)
  int64_t out = 0, out_m = 0;   // gather offsets (entries, mirrored entries)
  int64_t err_line = -1;        // local 0-based line of the first error
  std::string err_msg;
  int64_t last_entry_line = -1; // local line of the last entry parsed
};

struct ParseCtx {
  int64_t n_rows, n_cols, n_entries;
  bool universal;
};

void parse_chunk(Chunk& c, const ParseCtx& X) {
  const char* p = c.b;
  Line l;
  Line tok[3];
  int64_t ln = 0;
  const size_t guess = (size_t)((c.e - c.b) / 12 + 16);
  c.row.reserve(guess);
  c.col.reserve(guess);
  c.val.reserve(guess);
  for (; next_line(p, c.e, X.universal, &l); ++ln) {
    strip(&l);
    if (l.b == l.e || *l.b == '%') continue;
    // (the "more than the declared" check needs global counts: done later)
    const int nt = split(l, tok, 3);
    if (nt != 3) {
      c.err_line = ln;
      c.err_msg = "entry must hold row col value";
      break;
    }
    int64_t i = 0, j = 0;
    bool bi = false, bj = false;
    if (!py_int(tok[0], &i, &bi, nullptr) || !py_int(tok[1], &j, &bj, nullptr)) {
      c.err_line = ln;
      c.err_msg = "bad coordinate";
      break;
    }
    if (bi || i < 1 || i > X.n_rows) {
      std::string si;
      py_int(tok[0], &i, &bi, &si);
      c.err_line = ln;
      c.err_msg = "row index " + si + " out of range";
      break;
    }
    if (bj || j < 1 || j > X.n_cols) {
      std::string sj;
      py_int(tok[1], &j, &bj, &sj);
      c.err_line = ln;
      c.err_msg = "column index " + sj + " out of range";
      break;
    }
    double v = 0.0;
    if (!py_float(tok[2], &v)) {
      c.err_line = ln;
      c.err_msg = "bad value " + py_repr(str(tok[2]));
      break;
    }
    c.row.push_back((int32_t)(i - 1));
    c.col.push_back((int32_t)(j - 1));
    c.n_off += i != j;
    c.val.push_back(v);
    c.last_entry_line = ln;
  }
  // count the rest of the lines too (global numbering of later chunks)
  for (; next_line(p, c.e, X.universal, &l);) ++ln;
  c.n_lines = ln;
}

// local line of the k-th (0-based) entry of a chunk
int64_t entry_line(const Chunk& c, int64_t k, bool universal) {
  const char* p = c.b;
  Line l;
  int64_t ln = 0, seen = 0;
  for (; next_line(p, c.e, universal, &l); ++ln) {
    strip(&l);
    if (l.b == l.e || *l.b == '%') continue;
    if (seen++ == k) return ln;
  }
  return ln;
}

struct ParseError {
  int64_t line;
  std::string msg;
};

int fail(ParseError* pe, int64_t line, const std::string& msg) {
  pe->line = line;
  pe->msg = msg;
  return set_error(PCG_EPARSE, ("line " + std::to_string(line) + ": " + msg).c_str());
}

int parse_document(const char* data, int64_t len, bool universal, pcg_mm* M, ParseError* pe) {
  const char* p = data;
  const char* end = data + len;
  Line l;
  if (!next_line(p, end, universal, &l)) return fail(pe, 1, "empty document");
  int64_t line_no = 1;
  {
    strip(&l);
    std::string h = str(l);
    for (char& c : h) c = (char)tolower((unsigned char)c);
    Line hl{h.data(), h.data() + h.size()};
    Line t[5];
    const int nt = split(hl, t, 5);
    if (nt < 5 || str(t[0]) != "%%matrixmarket") return fail(pe, 1, "missing %%MatrixMarket header");
    if (str(t[1]) != "matrix") return fail(pe, 1, "unsupported object " + py_repr(str(t[1])));
    if (str(t[2]) != "coordinate") return fail(pe, 1, "unsupported format " + py_repr(str(t[2])));
    if (str(t[3]) != "real") return fail(pe, 1, "unsupported field " + py_repr(str(t[3])));
    const std::string sym = str(t[4]);
    if (sym != "general" && sym != "symmetric")
      return fail(pe, 1, "unsupported symmetry " + py_repr(sym));
    M->n_coo = sym == "symmetric" ? -1 : 0;  // marker until sized
  }
  const bool symmetric = M->n_coo == -1;
  // size line: first non-comment, non-blank line after the header
  int64_t size_no = -1;
  Line size_text{};
  while (next_line(p, end, universal, &l)) {
    ++line_no;
    strip(&l);
    if (l.b == l.e || *l.b == '%') continue;
    size_no = line_no;
    size_text = l;
    break;
  }
  if (size_no < 0) return fail(pe, 2, "missing size line");
  Line t[3];
  if (split(size_text, t, 3) != 3) return fail(pe, size_no, "size line must hold rows cols entries");
  int64_t dims[3];
  for (int k = 0; k < 3; ++k) {
    bool big = false;
    std::string norm;
    if (!py_int(t[k], &dims[k], &big, &norm))
      return fail(pe, size_no, "size line must hold three integers");
    if (big) return set_error(PCG_ERANGE, "Matrix Market size exceeds int64");
  }
  const int64_t n_rows = dims[0], n_cols = dims[1], n_entries = dims[2];
  if (n_rows <= 0 || n_cols <= 0 || n_entries <= 0) return fail(pe, size_no, "empty matrix");
  if (symmetric && n_rows != n_cols) return fail(pe, size_no, "symmetric matrix must be square");
  if (n_rows >= (1LL << 31) || n_cols >= (1LL << 31) ||
      (double)n_rows * (double)n_cols >= 9.2e18)
    return set_error(PCG_ERANGE, "Matrix Market: dimensions beyond the supported 2^31 rows/cols");

  // body: one chunk per thread, split after a '\n'
  const unsigned hw = std::max(1u, std::min(std::thread::hardware_concurrency(), 32u));
  const int64_t body = end - p;
  const int T = (int)std::max<int64_t>(1, std::min<int64_t>(hw, body / (1 << 20)));
  std::vector<Chunk> ch(T);
  const char* cur = p;
  for (int k = 0; k < T; ++k) {
    const char* stop = k == T - 1 ? end : std::max(cur, p + body * (k + 1) / T);
    if (k < T - 1) {
      while (stop < end && *stop != '\n') ++stop;
      if (stop < end) ++stop;
    }
    ch[k].b = cur;
    ch[k].e = stop;
    cur = stop;
  }
  const ParseCtx X{n_rows, n_cols, n_entries, universal};
  {
    std::vector<std::thread> th;
    for (int k = 1; k < T; ++k) th.emplace_back([&, k] { parse_chunk(ch[k], X); });
    parse_chunk(ch[0], X);
    for (auto& x : th) x.join();
  }
  // errors in document order; entry-count checks with global counts
  int64_t base = line_no;  // global line number of chunk line 0 is base + 1
  int64_t count = 0, last_no = size_no;
  for (int k = 0; k < T; ++k) {
    const Chunk& c = ch[k];
    const int64_t got = (int64_t)c.val.size();
    if (count + got > n_entries || (c.err_line >= 0 && count + got == n_entries)) {
      // the (n_entries+1)-th entry line raises before anything after it
      const int64_t kth = n_entries - count;
      const int64_t ln = kth < got ? entry_line(c, kth, universal) : c.err_line;
      return fail(pe, base + 1 + ln,
                  "more than the declared " + std::to_string(n_entries) + " entries");
    }
    if (c.err_line >= 0) return fail(pe, base + 1 + c.err_line, c.err_msg);
    count += got;
    if (c.last_entry_line >= 0) last_no = base + 1 + c.last_entry_line;
    base += c.n_lines;
  }
  if (count != n_entries)
    return fail(pe, last_no + 1, "expected " + std::to_string(n_entries) + " entries, found " +
                                     std::to_string(count));
  // gather (document order), symmetric: mirrored off-diagonals appended
  // after all entries; one thread per chunk at precomputed offsets
  M->n_rows = n_rows;
  M->n_cols = n_cols;
  int64_t n_off = 0, o = 0;
  for (auto& c : ch) {
    c.out = o;
    o += (int64_t)c.val.size();
  }
  for (auto& c : ch) {
    c.out_m = o + n_off;
    if (symmetric) n_off += c.n_off;
  }
  M->n_coo = count + n_off;
  M->key.resize(M->n_coo);
  M->val.resize(M->n_coo);
  auto gather = [&](Chunk& c) {
    int64_t* key = M->key.data();
    double* val = M->val.data();
    int64_t om = c.out_m;
    for (size_t q = 0; q < c.val.size(); ++q) {
      const int64_t r = c.row[q], cc = c.col[q];
      key[c.out + q] = r * n_cols + cc;
      val[c.out + q] = c.val[q];
      if (symmetric && r != cc) {
        key[om] = cc * n_cols + r;
        val[om] = c.val[q];
        ++om;
      }
    }
    std::vector<int32_t>().swap(c.row);
    std::vector<int32_t>().swap(c.col);
    std::vector<double>().swap(c.val);
  };
  {
    std::vector<std::thread> th;
    for (int k = 1; k < T; ++k) th.emplace_back([&, k] { gather(ch[k]); });
    gather(ch[0]);
    for (auto& x : th) x.join();
  }
  return PCG_OK;
}

// ---- device COO -> CSR ------------------------------------------------------
__global__ void seg_heads_kernel(int64_t n, const unsigned long long* key, int* head) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    head[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}

__global__ void seg_starts_kernel(int64_t n, const int* head, const int* seg, int64_t* start) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (head[i]) start[seg[i] - 1] = i;
}

// numpy's pairwise_sum (float64): what np.add.reduceat applies to a
// segment after its first element (sparse.py:316 sums duplicates that way):
// < 8 terms sequentially from 0.0, <= 128 eight interleaved accumulators,
// otherwise the two halves (split at a multiple of 8).
__device__ double np_pairwise(const double* a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, a[i]);
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i = 8;
    for (; i < n - n % 8; i += 8)
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(np_pairwise(a, n2), np_pairwise(a + n2, n - n2));
}

// one thread per distinct (row, col): duplicates (stable-sorted, so in
// document order) summed as the reference's np.add.reduceat does
__global__ void seg_sum_kernel(int64_t nnz, int64_t n, const int64_t* start,
                               const unsigned long long* key, const double* v, int64_t n_cols,
                               int* col, double* val, unsigned long long* row_count) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nnz;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = start[s], e = s + 1 < nnz ? start[s + 1] : n;
    const double acc = e - b > 1 ? __dadd_rn(v[b], np_pairwise(v + b + 1, e - b - 1)) : v[b];
    const int64_t kk = (int64_t)key[b];
    col[s] = (int)(kk % n_cols);
    val[s] = acc;
    atomicAdd(row_count + kk / n_cols, 1ull);
  }
}

template <typename RP>
__global__ void offsets_kernel(int64_t n_rows, const unsigned long long* incl, RP* rowptr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n_rows;
       i += (int64_t)gridDim.x * blockDim.x)
    rowptr[i] = i == 0 ? (RP)0 : (RP)incl[i - 1];
}

struct Dev {
  void* p = nullptr;
  ~Dev() { cudaFree(p); }
  bool alloc(size_t b) { return cudaMalloc(&p, b ? b : 16) == cudaSuccess; }
};

}  // namespace
}  // namespace pcg

using namespace pcg;

extern "C" {

static thread_local int64_t g_mm_err_line = 0;

int64_t pipecg_b200_mm_error_line(void) { return g_mm_err_line; }

int pipecg_b200_mm_parse(const char* data, int64_t len, int universal_newlines, pcg_mm** out) {
  if (!out || (len > 0 && !data) || len < 0) return set_error(PCG_EINVAL, "mm_parse: bad arguments");
  *out = nullptr;
  g_mm_err_line = 0;
  pcg_mm* M = new pcg_mm();
  ParseError pe{0, ""};
  const int rc = parse_document(data, len, universal_newlines != 0, M, &pe);
  if (rc) {
    g_mm_err_line = pe.line;
    delete M;
    return rc;
  }
  *out = M;
  return PCG_OK;
}

int pipecg_b200_mm_read(const char* path, pcg_mm** out) {
  if (!path || !out) return set_error(PCG_EINVAL, "mm_read: bad arguments");
  FILE* f = fopen(path, "rb");
  if (!f) return set_error(PCG_EIO, (std::string("cannot open ") + path).c_str());
  std::vector<char> buf;
  fseek(f, 0, SEEK_END);
  const long sz = ftell(f);
  fseek(f, 0, SEEK_SET);
  buf.resize(sz > 0 ? (size_t)sz : 0);
  const size_t got = sz > 0 ? fread(buf.data(), 1, buf.size(), f) : 0;
  fclose(f);
  if (got != buf.size()) return set_error(PCG_EIO, (std::string("cannot read ") + path).c_str());
  return pipecg_b200_mm_parse(buf.data(), (int64_t)buf.size(), 1, out);
}

int pipecg_b200_mm_info(const pcg_mm* M, int64_t* n_rows, int64_t* n_cols, int64_t* n_coo) {
  if (!M) return set_error(PCG_EINVAL, "mm_info: null handle");
  if (n_rows) *n_rows = M->n_rows;
  if (n_cols) *n_cols = M->n_cols;
  if (n_coo) *n_coo = M->n_coo;
  return PCG_OK;
}

void pipecg_b200_mm_free(pcg_mm* M) { delete M; }

int pipecg_b200_mm_to_csr(const pcg_mm* M, int rp64, void* rowptr, int32_t* col, double* val,
                          int64_t* nnz_out, void* stream) {
  if (!M || !rowptr || !col || !val || !nnz_out) return set_error(PCG_EINVAL, "mm_to_csr: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = M->n_coo, n_rows = M->n_rows;
  *nnz_out = 0;
  if (n >= (1LL << 31) - 1) return set_error(PCG_ERANGE, "mm_to_csr: >= 2^31 entries on one device");
  Dev k_in, k_out, v_in, v_out, head, seg, start, cnt, incl, tmp;
  if (!k_in.alloc(n * 8) || !k_out.alloc(n * 8) || !v_in.alloc(n * 8) || !v_out.alloc(n * 8) ||
      !head.alloc(n * 4) || !seg.alloc(n * 4) || !start.alloc(n * 8) ||
      !cnt.alloc(n_rows * 8) || !incl.alloc(n_rows * 8))
    return set_error(PCG_ENOMEM, "mm_to_csr: device workspace");
  int rc = pipecg_b200_h2d(k_in.p, M->key.data(), n, PCG_H2D_COPY64, st);
  if (!rc) rc = pipecg_b200_h2d(v_in.p, M->val.data(), n, PCG_H2D_COPY64, st);
  if (rc) return rc;
  int bits = 1;
  while (bits < 64 && ((unsigned long long)M->n_rows * (unsigned long long)M->n_cols) >> bits) ++bits;
  auto* ki = static_cast<unsigned long long*>(k_in.p);
  auto* ko = static_cast<unsigned long long*>(k_out.p);
  auto* vi = static_cast<double*>(v_in.p);
  auto* vo = static_cast<double*>(v_out.p);
  size_t b1 = 0, b2 = 0, b3 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, b1, ki, ko, vi, vo, n, 0, bits, st);  // stable
  cub::DeviceScan::InclusiveSum(nullptr, b2, static_cast<int*>(head.p), static_cast<int*>(seg.p), n, st);
  cub::DeviceScan::InclusiveSum(nullptr, b3, static_cast<unsigned long long*>(cnt.p),
                                static_cast<unsigned long long*>(incl.p), n_rows, st);
  if (!tmp.alloc(std::max({b1, b2, b3}))) return set_error(PCG_ENOMEM, "mm_to_csr: sort workspace");
  size_t bt = std::max({b1, b2, b3});
  cub::DeviceRadixSort::SortPairs(tmp.p, bt, ki, ko, vi, vo, n, 0, bits, st);
  const unsigned g = elementwise_grid(n);
  seg_heads_kernel<<<g, 256, 0, st>>>(n, ko, static_cast<int*>(head.p));
  bt = std::max({b1, b2, b3});
  cub::DeviceScan::InclusiveSum(tmp.p, bt, static_cast<int*>(head.p), static_cast<int*>(seg.p), n, st);
  int nnz = 0;
  cudaMemcpyAsync(&nnz, static_cast<int*>(seg.p) + n - 1, sizeof(int), cudaMemcpyDeviceToHost, st);
  rc = cuda_status(cudaStreamSynchronize(st), "mm_to_csr sort");
  if (rc) return rc;
  seg_starts_kernel<<<g, 256, 0, st>>>(n, static_cast<int*>(head.p), static_cast<int*>(seg.p),
                                       static_cast<int64_t*>(start.p));
  cudaMemsetAsync(cnt.p, 0, n_rows * 8, st);
  seg_sum_kernel<<<elementwise_grid(nnz), 256, 0, st>>>(
      nnz, n, static_cast<int64_t*>(start.p), ko, vo, M->n_cols, col, val,
      static_cast<unsigned long long*>(cnt.p));
  bt = std::max({b1, b2, b3});
  cub::DeviceScan::InclusiveSum(tmp.p, bt, static_cast<unsigned long long*>(cnt.p),
                                static_cast<unsigned long long*>(incl.p), n_rows, st);
  if (rp64)
    offsets_kernel<long long><<<elementwise_grid(n_rows + 1), 256, 0, st>>>(
        n_rows, static_cast<unsigned long long*>(incl.p), static_cast<long long*>(rowptr));
  else
    offsets_kernel<int><<<elementwise_grid(n_rows + 1), 256, 0, st>>>(
        n_rows, static_cast<unsigned long long*>(incl.p), static_cast<int*>(rowptr));
  rc = cuda_status(cudaStreamSynchronize(st), "mm_to_csr");
  if (rc) return rc;
  *nnz_out = nnz;
  return PCG_OK;
}

}  // extern "C"
