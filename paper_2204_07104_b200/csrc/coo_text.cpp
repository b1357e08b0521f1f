// coo_text.cpp -- multi-threaded reader of the reference's COO text format
// (load_coo, coo.py:90-148), SURVEY 8f row 1.
//
// The reference parses line by line in Python (~1 us per nonzero: minutes at
// 99M-1e9 nonzeros).  Here the file is memory-mapped, cut into T chunks at
// line terminators, and each thread tokenises its chunk with std::from_chars
// into per-chunk buffers; the caller then receives the arrays in file order.
// The accepted language and every error mirror the reference's:
//   * lines end at \n, \r or \r\n (Python's universal newlines, so line
//     numbers agree); blank lines are skipped; after stripping, a line that
//     starts with '#' is a comment, and "# dims: d_1 .. d_N" (case-insensitive
//     "dims:") sets the dims header (the last one wins; "bad dims header" if
//     a token is not an int);
//   * the first data line fixes the width (>= 3 tokens, else "need at least
//     2 indices and a value"); then per line, in this order: "expected K
//     tokens, got M", "unparseable token" (Python int()/float() grammar:
//     sign, '_' between digits, inf/infinity/nan), "index below base B",
//     "non-finite value";
//   * the error raised is the earliest one in file order, with its 1-based
//     line number, exactly as the sequential reader would report it.
// Whitespace is the ASCII set Python's str.split() uses (space, \t, \v, \f,
// \x1c-\x1f); non-ASCII bytes are token characters.  Indices that do not fit
// int64 are reported as an overflow (the reference's np.asarray raises
// OverflowError there).
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

namespace sptk {
void set_error(const char* fmt, ...);
}

namespace {

enum { kOk = 0, kFormat = 1, kOs = 2, kOverflow = 3 };

inline bool is_ws(unsigned char c) {
  return c == ' ' || c == '\t' || c == '\v' || c == '\f' || (c >= 0x1c && c <= 0x1f);
}
inline bool is_eol(unsigned char c) { return c == '\n' || c == '\r'; }

// Python int(): [sign] digit (['_'] digit)*  (leading zeros allowed).
// Returns 0 ok, 1 syntax error, 2 overflow.
int parse_int(const char* b, const char* e, int64_t* out) {
  if (b == e) return 1;
  bool neg = false;
  if (*b == '+' || *b == '-') {
    neg = *b == '-';
    ++b;
  }
  if (b == e || *b < '0' || *b > '9') return 1;
  unsigned __int128 v = 0;
  bool prev_digit = false, big = false;
  for (; b < e; ++b) {
    char c = *b;
    if (c >= '0' && c <= '9') {
      if (!big) {
        v = v * 10 + unsigned(c - '0');
        if (v > (unsigned __int128)1 << 64) big = true;
      }
      prev_digit = true;
    } else if (c == '_' && prev_digit && b + 1 < e && b[1] >= '0' && b[1] <= '9') {
      prev_digit = false;
    } else {
      return 1;
    }
  }
  const unsigned __int128 lim = neg ? ((unsigned __int128)1 << 63) : (((unsigned __int128)1 << 63) - 1);
  if (big || v > lim) return 2;
  *out = neg ? (int64_t)(-(__int128)v) : (int64_t)v;
  return 0;
}

bool ieq(const char* b, const char* e, const char* lit) {
  size_t n = strlen(lit);
  if ((size_t)(e - b) != n) return false;
  for (size_t i = 0; i < n; ++i) {
    char c = b[i];
    if (c >= 'A' && c <= 'Z') c = char(c - 'A' + 'a');
    if (c != lit[i]) return false;
  }
  return true;
}

// Python float(): [sign] (inf | infinity | nan | decimal), decimal =
// (digitpart ['.' [digitpart]] | '.' digitpart) [('e'|'E') [sign] digitpart],
// digitpart = digit (['_'] digit)*.  Correctly rounded (from_chars), as
// Python's float() is.
bool parse_float(const char* b, const char* e, double* out) {
  if (b == e) return false;
  bool neg = false;
  const char* p = b;
  if (*p == '+' || *p == '-') {
    neg = *p == '-';
    ++p;
  }
  if (ieq(p, e, "inf") || ieq(p, e, "infinity")) {
    *out = neg ? -INFINITY : INFINITY;
    return true;
  }
  if (ieq(p, e, "nan")) {
    *out = NAN;
    return true;
  }
  char stackbuf[128];
  std::string heap;
  char* buf = stackbuf;
  size_t cap = sizeof(stackbuf);
  if ((size_t)(e - b) + 1 > cap) {
    heap.resize((size_t)(e - b) + 1);
    buf = &heap[0];
    cap = heap.size();
  }
  size_t n = 0;
  if (neg) buf[n++] = '-';
  // digitpart scanner: copies digits (dropping single '_' between digits)
  auto digits = [&](const char*& q) -> int {
    int cnt = 0;
    while (q < e) {
      if (*q >= '0' && *q <= '9') {
        buf[n++] = *q++;
        ++cnt;
      } else if (*q == '_' && cnt > 0 && q + 1 < e && q[1] >= '0' && q[1] <= '9') {
        ++q;
      } else {
        break;
      }
    }
    return cnt;
  };
  int int_digits = digits(p);
  int frac_digits = 0;
  if (p < e && *p == '.') {
    buf[n++] = *p++;
    frac_digits = digits(p);
  }
  if (int_digits == 0 && frac_digits == 0) return false;
  if (p < e && (*p == 'e' || *p == 'E')) {
    buf[n++] = 'e';
    ++p;
    if (p < e && (*p == '+' || *p == '-')) buf[n++] = *p++;
    if (digits(p) == 0) return false;
  }
  if (p != e) return false;
  double v = 0.0;
  auto r = std::from_chars(buf, buf + n, v, std::chars_format::general);
  if (r.ec == std::errc::result_out_of_range) {
    // from_chars leaves v untouched on range errors; Python rounds to
    // +-inf / +-0 / a subnormal like strtod (correctly rounded in glibc)
    buf[n] = 0;
    v = strtod(buf, nullptr);
  } else if (r.ec != std::errc() || r.ptr != buf + n) {
    return false;
  }
  *out = v;
  return true;
}

struct Err {
  int64_t line = -1;  // local (chunk-relative, 1-based) line of the first error
  int code = kOk;
  std::string msg;  // without the "line N: " prefix
};

struct Chunk {
  const char* b = nullptr;
  const char* e = nullptr;
  int64_t lines = 0;  // line terminators (a final unterminated line counts 1)
  std::vector<int64_t> idx;
  std::vector<double> val;
  std::vector<int64_t> mx;  // per-mode max index
  int64_t overflow_line = 0;  // first line whose index does not fit int64 (reported last)
  bool has_dims = false;
  int64_t dims_line = 0;
  std::vector<int64_t> dims;
  Err err;
};

struct Parsed {
  int order = 0;
  int64_t nnz = 0;
  std::vector<Chunk> chunks;
  std::vector<int64_t> dims;
  bool dims_from_header = false;
};

// Process one chunk: every line inside [b, e).  `width` = tokens of the first
// data line of the file (0 if none), `first_data` = its address.
void parse_chunk(Chunk& c, int width, const char* first_data, int64_t base) {
  const int order = width - 1;
  if (order > 0) c.mx.assign(order, -1);
  std::vector<const char*> tb, te;
  tb.reserve(16);
  te.reserve(16);
  const char* p = c.b;
  int64_t line = 0;
  auto fail = [&](int code, std::string msg) {
    if (c.err.code == kOk) {
      c.err.line = line;
      c.err.code = code;
      c.err.msg = std::move(msg);
    }
  };
  while (p < c.e && c.err.code == kOk) {
    const char* ls = p;
    while (p < c.e && !is_eol((unsigned char)*p)) ++p;
    const char* le = p;
    if (p < c.e) {
      if (*p == '\r' && p + 1 < c.e && p[1] == '\n') ++p;
      ++p;
    }
    ++line;
    // strip (the terminator is already excluded)
    while (ls < le && is_ws((unsigned char)*ls)) ++ls;
    while (le > ls && is_ws((unsigned char)le[-1])) --le;
    if (ls == le) continue;
    if (*ls == '#') {
      const char* q = ls + 1;
      while (q < le && is_ws((unsigned char)*q)) ++q;
      if (le - q >= 5 && ieq(q, q + 5, "dims:")) {
        q += 5;
        std::vector<int64_t> d;
        while (q < le) {
          while (q < le && is_ws((unsigned char)*q)) ++q;
          if (q >= le) break;
          const char* s = q;
          while (q < le && !is_ws((unsigned char)*q)) ++q;
          int64_t v = 0;
          int rc = parse_int(s, q, &v);
          if (rc == 1) {
            fail(kFormat, "bad dims header");
            break;
          }
          if (rc == 2) {
            fail(kOverflow, "dims header value does not fit int64");
            break;
          }
          d.push_back(v);
        }
        if (c.err.code == kOk) {
          c.has_dims = true;
          c.dims_line = line;
          c.dims = std::move(d);
        }
      }
      continue;
    }
    tb.clear();
    te.clear();
    for (const char* q = ls; q < le;) {
      while (q < le && is_ws((unsigned char)*q)) ++q;
      if (q >= le) break;
      tb.push_back(q);
      while (q < le && !is_ws((unsigned char)*q)) ++q;
      te.push_back(q);
    }
    const int ntok = (int)tb.size();
    if (ls == first_data && width < 3) {
      fail(kFormat, "need at least 2 indices and a value");
      break;
    }
    if (ntok != width) {
      fail(kFormat, "expected " + std::to_string(width) + " tokens, got " + std::to_string(ntok));
      break;
    }
    int64_t ix[64];
    bool ok = true;
    bool over = false;
    for (int n = 0; n < order; ++n) {
      int rc = parse_int(tb[n], te[n], &ix[n]);
      if (rc == 1) ok = false;
      if (rc == 2) over = true;
    }
    double v = 0.0;
    if (!parse_float(tb[order], te[order], &v)) ok = false;
    if (!ok) {
      fail(kFormat, "unparseable token");
      break;
    }
    if (over) {
      // Python keeps the big int: a huge negative one is "below base" now; a
      // huge positive one passes the line checks and only fails the final
      // np.asarray (OverflowError after the whole file parsed)
      bool neg_big = false;
      for (int n = 0; n < order; ++n) {
        int64_t tmp;
        if (parse_int(tb[n], te[n], &tmp) == 2) {
          if (*tb[n] == '-') neg_big = true;
          ix[n] = base;
        }
      }
      if (neg_big) {
        fail(kFormat, "index below base " + std::to_string(base));
        break;
      }
      if (c.overflow_line == 0) c.overflow_line = line;
    }
    bool below = false;
    for (int n = 0; n < order; ++n) below |= ix[n] < base;
    if (below) {
      fail(kFormat, "index below base " + std::to_string(base));
      break;
    }
    if (!std::isfinite(v)) {
      fail(kFormat, "non-finite value");
      break;
    }
    for (int n = 0; n < order; ++n) {
      int64_t k = ix[n] - base;
      c.idx.push_back(k);
      if (k > c.mx[n]) c.mx[n] = k;
    }
    c.val.push_back(v);
  }
  // line count of the whole chunk (for the global numbering)
  if (c.err.code == kOk) {
    c.lines = line;
  } else {
    int64_t n = 0;
    for (const char* q = c.b; q < c.e; ++q) {
      if (*q == '\n' || (*q == '\r' && !(q + 1 < c.e && q[1] == '\n'))) ++n;
    }
    if (c.e > c.b && !is_eol((unsigned char)c.e[-1])) ++n;
    c.lines = n;
  }
}

// Start of the line after the terminator at or after g.
const char* next_line(const char* g, const char* b, const char* e) {
  if (g <= b) return b;
  if (g >= e) return e;
  // g inside "\r\n" (just after the \r): the line already ended
  if (*g == '\n' && g[-1] == '\r') return g + 1;
  while (g < e && !is_eol((unsigned char)*g)) ++g;
  if (g >= e) return e;
  if (*g == '\r' && g + 1 < e && g[1] == '\n') return g + 2;
  return g + 1;
}

}  // namespace

extern "C" {

// Parse `path`; on success *handle owns the parsed arrays (sptk_coo_text_take
// copies them out and frees it).  Returns 0, 1 (format error: message
// "line N: ..."; N = 0 for whole-file errors), 2 (OS error) or 3 (overflow).
int sptk_coo_text_parse(const char* path, int index_base, int threads, void** handle, int64_t* nnz,
                        int* order) {
  *handle = nullptr;
  int fd = open(path, O_RDONLY);
  if (fd < 0) {
    sptk::set_error("%s: %s", path, strerror(errno));
    return kOs;
  }
  struct stat st;
  if (fstat(fd, &st) != 0) {
    sptk::set_error("%s: %s", path, strerror(errno));
    close(fd);
    return kOs;
  }
  size_t size = (size_t)st.st_size;
  const char* data = nullptr;
  void* map = nullptr;
  if (size > 0) {
    map = mmap(nullptr, size, PROT_READ, MAP_PRIVATE, fd, 0);
    if (map == MAP_FAILED) {
      sptk::set_error("%s: mmap: %s", path, strerror(errno));
      close(fd);
      return kOs;
    }
    madvise(map, size, MADV_SEQUENTIAL | MADV_WILLNEED);
    data = (const char*)map;
  }
  close(fd);
  const char* b = data;
  const char* e = data + size;

  // first data line (sequential; comments before it are handled by the
  // chunk parsers in file order)
  int width = 0;
  const char* first_data = nullptr;
  for (const char* p = b; p < e;) {
    const char* ls = p;
    while (p < e && !is_eol((unsigned char)*p)) ++p;
    const char* le = p;
    if (p < e) {
      if (*p == '\r' && p + 1 < e && p[1] == '\n') ++p;
      ++p;
    }
    while (ls < le && is_ws((unsigned char)*ls)) ++ls;
    while (le > ls && is_ws((unsigned char)le[-1])) --le;
    if (ls == le || *ls == '#') continue;
    first_data = ls;
    for (const char* q = ls; q < le;) {
      while (q < le && is_ws((unsigned char)*q)) ++q;
      if (q >= le) break;
      ++width;
      while (q < le && !is_ws((unsigned char)*q)) ++q;
    }
    break;
  }
  if (width - 1 > 64) {
    sptk::set_error("line 0: tensor order %d above the supported 64", width - 1);
    if (map) munmap(map, size);
    return kFormat;
  }

  int T = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
  if (T < 1) T = 1;
  if (T > 256) T = 256;
  if (size < ((size_t)1 << 20)) T = 1;
  auto* P = new Parsed();
  P->chunks.resize(T);
  const char* prev = b;
  for (int i = 0; i < T; ++i) {
    const char* end = (i + 1 == T) ? e : next_line(b + (size * (i + 1)) / T, b, e);
    if (end < prev) end = prev;
    P->chunks[i].b = prev;
    P->chunks[i].e = end;
    prev = end;
  }
  {
    std::vector<std::thread> th;
    for (int i = 1; i < T; ++i)
      th.emplace_back(parse_chunk, std::ref(P->chunks[i]), width, first_data, (int64_t)index_base);
    parse_chunk(P->chunks[0], width, first_data, (int64_t)index_base);
    for (auto& t : th) t.join();
  }
  if (map) munmap(map, size);
  for (auto& c : P->chunks) {  // the chunk pointers are dangling from here on
    c.b = c.e = nullptr;
  }
  // earliest error in file order
  int64_t line0 = 0;
  for (auto& c : P->chunks) {
    if (c.err.code != kOk) {
      sptk::set_error("line %lld: %s", (long long)(line0 + c.err.line), c.err.msg.c_str());
      int code = c.err.code;
      delete P;
      return code;
    }
    line0 += c.lines;
  }
  line0 = 0;
  for (auto& c : P->chunks) {
    if (c.overflow_line) {
      sptk::set_error("line %lld: index does not fit int64", (long long)(line0 + c.overflow_line));
      delete P;
      return kOverflow;
    }
    line0 += c.lines;
  }
  const int N = width - 1;
  int64_t total = 0;
  for (auto& c : P->chunks) total += (int64_t)c.val.size();
  if (total == 0) {
    sptk::set_error("line 0: no entries in file");
    delete P;
    return kFormat;
  }
  P->order = N;
  P->nnz = total;
  // dims: the last header in file order, else max index + 1
  for (auto& c : P->chunks)
    if (c.has_dims) {
      P->dims = c.dims;
      P->dims_from_header = true;
    }
  if (P->dims_from_header) {
    if ((int)P->dims.size() != N) {
      sptk::set_error("line 0: dims header length does not match entry order");
      delete P;
      return kFormat;
    }
  } else {
    P->dims.assign(N, 0);
    for (auto& c : P->chunks)
      for (int n = 0; n < N && !c.mx.empty(); ++n)
        if (c.mx[n] + 1 > P->dims[n]) P->dims[n] = c.mx[n] + 1;
  }
  *handle = P;
  *nnz = total;
  *order = N;
  return kOk;
}

// dims (order entries) and whether they came from a "# dims:" header.
int sptk_coo_text_dims(void* handle, int64_t* dims, int* from_header) {
  auto* P = (Parsed*)handle;
  for (int n = 0; n < P->order; ++n) dims[n] = P->dims[n];
  *from_header = P->dims_from_header ? 1 : 0;
  return 0;
}

// Copy the parsed entries (file order) into indices [nnz, order] (int64,
// C order, 0-based) and values [nnz] (float64), then free the handle.
int sptk_coo_text_take(void* handle, int64_t* indices, double* values, int threads) {
  auto* P = (Parsed*)handle;
  const int N = P->order;
  std::vector<int64_t> off(P->chunks.size() + 1, 0);
  for (size_t i = 0; i < P->chunks.size(); ++i) off[i + 1] = off[i] + (int64_t)P->chunks[i].val.size();
  auto copy = [&](size_t i) {
    Chunk& c = P->chunks[i];
    if (!c.val.empty()) {
      memcpy(indices + off[i] * N, c.idx.data(), c.idx.size() * sizeof(int64_t));
      memcpy(values + off[i], c.val.data(), c.val.size() * sizeof(double));
    }
    std::vector<int64_t>().swap(c.idx);
    std::vector<double>().swap(c.val);
  };
  int T = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
  if (T < 1) T = 1;
  std::vector<std::thread> th;
  for (int t = 0; t < T && (size_t)t < P->chunks.size(); ++t)
    th.emplace_back([&, t] {
      for (size_t i = t; i < P->chunks.size(); i += T) copy(i);
    });
  for (auto& x : th) x.join();
  delete P;
  return 0;
}

void sptk_coo_text_free(void* handle) { delete (Parsed*)handle; }

}  // extern "C"
