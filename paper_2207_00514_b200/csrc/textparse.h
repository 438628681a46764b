// textparse.h -- the reference's CSV readers (data.py:148-198 read_points,
// 225-257 read_edges) parsed on all host threads.
//
// The reference iterates the lines of a text-mode file (universal newlines:
// "\n", "\r\n" and a lone "\r" all end a line), strips each one, skips blank
// lines, splits on ',' and converts every field with Python's int() / float().
// Here the buffer is cut into blocks at line ends; one pass counts the rows
// and line ends of every block, a scan turns the counts into output offsets
// and line numbers, and a second pass parses every block in place.
//
// Only the plain ASCII spellings are converted natively: optional sign and
// digits for an endpoint, sign / digits / point / exponent for a coordinate or
// weight (std::from_chars: correctly rounded, as float() is).  Anything else --
// a non-ASCII byte, an underscore, "inf", an overflow, a negative endpoint, a
// wrong field count -- stops the parse at that line and hands it back to the
// caller, which applies the reference's own rules to that one line (raising
// its ParseError, or accepting a spelling like "1_000") and resumes after it.
// The earliest such line over all blocks wins, so errors are reported for the
// same line as the reference's sequential loop.
#pragma once
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace emst_io {

struct ParseStop {
  int64_t rows = 0;        // rows written before the stop (or all rows)
  int64_t line = -1;       // 1-based line number of the line handed back, -1 when none
  int64_t begin = 0;       // its byte range, line terminator excluded
  int64_t end = 0;
  int64_t next = 0;        // where to resume: just past its terminator
  int32_t width = 0;       // fields per row (points: detected from the first row)
};

// Python's str.isspace() over ASCII: \t \n \v \f \r, \x1c-\x1f and space.
inline bool py_space(unsigned char c) { return c == ' ' || (c >= 9 && c <= 13) || (c >= 0x1c && c <= 0x1f); }

// End of the line starting at p (first terminator byte or `end`), and the start of the next line.
inline const char* line_end(const char* p, const char* end, const char** next) {
  const char* q = p;
  while (q < end && *q != '\n' && *q != '\r') ++q;
  const char* nx = q;
  if (nx < end) nx += (*nx == '\r' && nx + 1 < end && nx[1] == '\n') ? 2 : 1;
  *next = nx;
  return q;
}

inline void strip(const char*& a, const char*& b) {
  while (a < b && py_space((unsigned char)*a)) ++a;
  while (b > a && py_space((unsigned char)b[-1])) --b;
}

inline bool ascii_only(const char* a, const char* b) {
  for (; a < b; ++a)
    if ((unsigned char)*a >= 0x80) return false;
  return true;
}

// [+-]?[0-9]{1,18} -> v >= 0 (a negative endpoint is the caller's error to report)
inline bool parse_index(const char* a, const char* b, int64_t* v) {
  strip(a, b);
  bool neg = false;
  if (a < b && (*a == '+' || *a == '-')) neg = *a++ == '-';
  if (a == b || b - a > 18) return false;
  int64_t x = 0;
  for (const char* p = a; p < b; ++p) {
    if (*p < '0' || *p > '9') return false;
    x = x * 10 + (*p - '0');
  }
  if (neg && x != 0) return false;
  *v = x;
  return true;
}

// [+-]?(digits[.digits?]|.digits)([eE][+-]?digits)? -> a finite double
inline bool parse_real(const char* a, const char* b, double* v) {
  strip(a, b);
  const char* p = a;
  if (p < b && (*p == '+' || *p == '-')) ++p;
  const char* m = p;
  int digits = 0;
  while (p < b && *p >= '0' && *p <= '9') ++p, ++digits;
  if (p < b && *p == '.') {
    ++p;
    while (p < b && *p >= '0' && *p <= '9') ++p, ++digits;
  }
  if (!digits) return false;
  if (p < b && (*p == 'e' || *p == 'E')) {
    ++p;
    if (p < b && (*p == '+' || *p == '-')) ++p;
    const char* e = p;
    while (p < b && *p >= '0' && *p <= '9') ++p;
    if (p == e) return false;
  }
  if (p != b) return false;
  double x = 0.0;
  auto r = std::from_chars(m, b, x, std::chars_format::general);
  if (r.ec != std::errc() || r.ptr != b || !std::isfinite(x)) return false;   // (over/underflow: the caller's rules)
  *v = *a == '-' ? -x : x;
  return true;
}

// One row into slot `row` of the outputs; false hands the line back.
// edges: a = int64 (m, 2), b = f64 weights; points: a = f32 (n, width).
inline bool parse_row(const char* a, const char* b, bool edges, int width, int64_t row, void* out_a, void* out_b) {
  if (!ascii_only(a, b)) return false;
  const char* f[3];
  const char* g[3];
  int k = 0;
  const char* s = a;
  for (const char* p = a;; ++p) {
    if (p == b || *p == ',') {
      if (k == 3) return false;
      f[k] = s;
      g[k] = p;
      ++k;
      s = p + 1;
      if (p == b) break;
    }
  }
  if (k != (edges ? 3 : width)) return false;
  if (edges) {
    int64_t u, v;
    double w;
    if (!parse_index(f[0], g[0], &u) || !parse_index(f[1], g[1], &v) || !parse_real(f[2], g[2], &w)) return false;
    reinterpret_cast<int64_t*>(out_a)[2 * row] = u;
    reinterpret_cast<int64_t*>(out_a)[2 * row + 1] = v;
    reinterpret_cast<double*>(out_b)[row] = w;
  } else {
    float* o = reinterpret_cast<float*>(out_a) + row * width;
    for (int j = 0; j < width; ++j) {
      double x;
      if (!parse_real(f[j], g[j], &x)) return false;
      o[j] = (float)x;   // np.asarray(rows, dtype=float32): round to nearest
    }
  }
  return true;
}

struct Block {
  const char* a;
  const char* b;
  int64_t rows = 0, lines = 0;
};

// Block boundaries just after a '\n' (so "\r\n" is never split), about `parts` blocks.
inline std::vector<Block> cut_blocks(const char* a, const char* b, int parts) {
  std::vector<Block> out;
  const int64_t len = b - a;
  const char* s = a;
  for (int t = 1; t <= parts && s < b; ++t) {
    const char* e = t == parts ? b : std::max(s, a + len * t / parts);
    if (e < b) {
      const char* nl = (const char*)memchr(e, '\n', (size_t)(b - e));
      e = nl ? nl + 1 : b;
    }
    if (e > s) out.push_back({s, e});
    s = e;
  }
  return out;
}

template <class F>
void for_blocks(std::vector<Block>& blocks, F fn) {
  std::vector<std::thread> pool;
  for (size_t i = 1; i < blocks.size(); ++i) pool.emplace_back([&, i] { fn(blocks[i]); });
  if (!blocks.empty()) fn(blocks[0]);
  for (auto& t : pool) t.join();
}

// Non-blank lines of [a, b).
inline int64_t count_rows(const char* a, const char* b) {
  auto blocks = cut_blocks(a, b, host_threads());
  for_blocks(blocks, [](Block& k) {
    const char* p = k.a;
    while (p < k.b) {
      const char* nx;
      const char* e = line_end(p, k.b, &nx);
      const char* s = p;
      strip(s, e);
      if (s < e) ++k.rows;
      p = nx;
    }
  });
  int64_t n = 0;
  for (auto& k : blocks) n += k.rows;
  return n;
}

// Parse [text + start, text + len) into rows [row0, cap) of the outputs; `line0` is the number of
// the first line.  points: width 0 detects it from the first non-blank line (2 or 3).
inline ParseStop parse_csv(const char* text, int64_t len, int64_t start, int64_t line0, int64_t row0, bool edges,
                           int width, void* out_a, void* out_b, int64_t cap) {
  ParseStop st;
  st.rows = row0;
  const char* a = text + start;
  const char* b = text + len;
  if (!edges && width == 0) {   // serial: the first non-blank line fixes the width
    int64_t line = line0;
    while (a < b) {
      const char* nx;
      const char* e = line_end(a, b, &nx);
      const char* s = a;
      strip(s, e);
      if (s < e) {
        int fields = 1;
        for (const char* p = s; p < e; ++p) fields += *p == ',';
        if ((fields != 2 && fields != 3) || !ascii_only(s, e)) {
          st.line = line;
          st.begin = a - text;
          st.end = line_end(a, b, &nx) - text;
          st.next = nx - text;
          return st;
        }
        width = fields;
        break;
      }
      a = nx;
      ++line;
    }
    line0 = line;
  }
  st.width = edges ? 3 : width;
  auto blocks = cut_blocks(a, b, host_threads());
  for_blocks(blocks, [](Block& k) {   // rows and line ends per block
    const char* p = k.a;
    while (p < k.b) {
      const char* nx;
      const char* e = line_end(p, k.b, &nx);
      const char* s = p;
      strip(s, e);
      if (s < e) ++k.rows;
      ++k.lines;
      p = nx;
    }
  });
  std::vector<int64_t> row_at(blocks.size()), line_at(blocks.size());
  int64_t r = row0, l = line0;
  for (size_t i = 0; i < blocks.size(); ++i) {
    row_at[i] = r;
    line_at[i] = l;
    r += blocks[i].rows;
    l += blocks[i].lines;
  }
  if (r > cap) {   // (the caller sized the outputs with count_rows over the same bytes)
    st.line = -2;
    return st;
  }
  std::vector<ParseStop> stops(blocks.size());
  for (size_t i = 0; i < blocks.size(); ++i) stops[i].rows = row_at[i];
  std::vector<int> idx(blocks.size());
  for (size_t i = 0; i < blocks.size(); ++i) idx[i] = (int)i;
  std::vector<std::thread> pool;
  auto work = [&](size_t i) {
    Block& k = blocks[i];
    ParseStop& s = stops[i];
    int64_t row = row_at[i], line = line_at[i];
    const char* p = k.a;
    while (p < k.b) {
      const char* nx;
      const char* e = line_end(p, k.b, &nx);
      const char* x = p;
      const char* y = e;
      strip(x, y);
      if (x < y) {
        if (!parse_row(x, y, edges, width, row, out_a, out_b)) {
          s.line = line;
          s.begin = p - text;
          s.end = e - text;
          s.next = nx - text;
          s.rows = row;
          return;
        }
        ++row;
      }
      ++line;
      p = nx;
    }
    s.rows = row;
  };
  for (size_t i = 1; i < blocks.size(); ++i) pool.emplace_back(work, i);
  if (!blocks.empty()) work(0);
  for (auto& t : pool) t.join();
  st.rows = r;
  for (size_t i = 0; i < blocks.size(); ++i)
    if (stops[i].line >= 0) {
      const int32_t w = st.width;
      st = stops[i];
      st.width = w;
      break;
    }
  return st;
}

}  // namespace emst_io
