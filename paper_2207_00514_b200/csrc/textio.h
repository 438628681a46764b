// textio.h -- host-side text formatting of edge lists and point clouds, byte
// for byte what the reference's Python writers produce (data.py:117-141, 222-235):
//   write_edges:  "%lld,%lld,%.17g\n" per edge   (f"{int(u)},{int(v)},{float(w):.17g}\n")
//   write_points: "%.9g" per coordinate, ',' separated, '\n' per row
//                 (",".join(f"{float(x):.9g}" for x in row))
// Python's 'g' formatting is C99 %g on a correctly rounded decimal expansion
// (PyOS_double_to_string); std::to_chars(general, precision) is specified as
// printf's %.*g and libstdc++ implements it exactly (Ryu printf), ~3x faster
// than snprintf, so the strings are identical.  The rows are split over host threads; every thread formats
// its contiguous block into its own buffer and the blocks are concatenated in
// order.  (the reference's Python loop takes minutes at
// 37M edges.)
#pragma once
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

namespace emst_io {

inline int host_threads() {
  const unsigned h = std::thread::hardware_concurrency();
  return h ? (int)std::min(h, 64u) : 1;
}

// Format rows [0, m) with fmt_row(i, char* out) -> bytes written (<= row_max),
// in parallel, into one contiguous string.
template <class F>
std::string format_rows(int64_t m, size_t row_max, F fmt_row) {
  const int T = (int)std::max<int64_t>(1, std::min<int64_t>(host_threads(), (m + 65535) / 65536));
  std::vector<std::string> parts(T);
  std::vector<std::thread> pool;
  for (int t = 0; t < T; ++t) {
    pool.emplace_back([&, t]() {
      const int64_t a = m * t / T, b = m * (t + 1) / T;
      std::string& s = parts[t];
      s.resize((size_t)(b - a) * row_max);
      char* p = &s[0];
      for (int64_t i = a; i < b; ++i) p += fmt_row(i, p);
      s.resize((size_t)(p - &s[0]));
    });
  }
  for (auto& th : pool) th.join();
  size_t total = 0;
  for (auto& s : parts) total += s.size();
  std::string out;
  out.reserve(total);
  for (auto& s : parts) out += s;
  return out;
}

inline char* put_i64(char* p, char* end, long long v) { return std::to_chars(p, end, v).ptr; }
inline char* put_g(char* p, char* end, double v, int prec) {
  return std::to_chars(p, end, v, std::chars_format::general, prec).ptr;
}

inline std::string format_edges(const int64_t* edges, const double* weights, int64_t m) {
  // two int64 (<= 20 chars each), a %.17g double (<= 24 chars), 2 commas, newline
  return format_rows(m, 72, [&](int64_t i, char* p) -> size_t {
    char* q = p;
    char* end = p + 72;
    q = put_i64(q, end, (long long)edges[2 * i]);
    *q++ = ',';
    q = put_i64(q, end, (long long)edges[2 * i + 1]);
    *q++ = ',';
    q = put_g(q, end, weights[i], 17);
    *q++ = '\n';
    return (size_t)(q - p);
  });
}

inline std::string format_points(const float* pts, int64_t n, int d) {
  // <= 3 coordinates of <= 16 chars (%.9g of a float), separators, newline
  return format_rows(n, 64, [&](int64_t i, char* p) -> size_t {
    char* q = p;
    for (int j = 0; j < d; ++j) {
      if (j) *q++ = ',';
      q = put_g(q, p + 64, (double)pts[i * d + j], 9);
    }
    *q++ = '\n';
    return (size_t)(q - p);
  });
}

}  // namespace emst_io
