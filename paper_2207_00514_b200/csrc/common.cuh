// common.cuh -- shared types and device helpers for the B200 EMST kernels.
//
// Layout conventions:
//   * slot      = position in Morton (Z) order; every per-point array is slot-indexed.
//   * perm[s]   = original point index of slot s (u32);  iperm = inverse.
//   * node ref  = int32: >= 0 internal node (Karras index), < 0 leaf slot ~ref.
//   * component = dense id in [0, c) per Boruvka round; MIXED = -1.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace emst {

constexpr int kMixed = -1;              // mst.py:57
constexpr int kStackCapacity = 64;      // bvh.py:36 STACK_CAPACITY
constexpr unsigned long long kNoBound = ~0ull;   // "+inf" for u64-bit-pattern mins

// One internal node's two children, fetched by a single 64-byte node visit.
// Leaf children carry their point as a degenerate box, so leaf distances need
// no second fetch.  Child labels are rewritten every Boruvka round.  The two
// children's coordinates are interleaved (left, right) so that every pair sits
// in an aligned register pair and both box tests run as packed f32x2 math:
// float k of child `side` is lo[k] at 2k + side and hi[k] at 2D + 2k + side.
struct __align__(16) Node3 {
  float4 a;   // lo.x L R, lo.y L R
  float4 b;   // lo.z L R, hi.x L R
  float4 c;   // hi.y L R, hi.z L R
  int4 ref;   // left ref, right ref, left label, right label
};
struct __align__(16) Node2 {
  float4 a;   // lo.x L R, lo.y L R
  float4 b;   // hi.x L R, hi.y L R
  int4 ref;
};

template <int D> struct NodeOf;
template <> struct NodeOf<2> { using type = Node2; };
template <> struct NodeOf<3> { using type = Node3; };

struct Box3 { float lo[3], hi[3]; };

// Per-component minimum outgoing edge, ordered by (w, u, v) with w the f64
// bit pattern (w >= 0, so bits order like values) and uv = u << 32 | v over
// original point indices (mst.py:62-89).  All-ones = "no edge yet".
struct __align__(16) EdgeKey {
  unsigned long long uv;
  unsigned long long w;
};

__device__ __forceinline__ bool key_less(unsigned long long w, unsigned long long uv,
                                         unsigned long long bw, unsigned long long buv) {
  return w < bw || (w == bw && uv < buv);
}

// Lexicographic 128-bit atomic min via the sm_90+ 16-byte CAS.  The first CAS
// expects the empty key (the common case for the first candidate of a
// component); a failed CAS returns the current key, and the loop only retries
// while ours is strictly smaller, so contended components rarely loop.
__device__ __forceinline__ void atomic_min_key(EdgeKey* addr, unsigned long long w, unsigned long long uv) {
  EdgeKey cur;
  cur.uv = ~0ull;
  cur.w = ~0ull;
  EdgeKey mine;
  mine.w = w;
  mine.uv = uv;
  while (key_less(w, uv, cur.w, cur.uv)) {
    EdgeKey old = atomicCAS(addr, cur, mine);
    if (old.w == cur.w && old.uv == cur.uv) return;
    cur = old;
  }
}

// Plain 16-byte store of a key (a component written by exactly one query).
__device__ __forceinline__ void store_key(EdgeKey* addr, unsigned long long w, unsigned long long uv) {
  asm volatile("st.global.v2.u64 [%0], {%1, %2};" :: "l"(addr), "l"(uv), "l"(w) : "memory");
}

// Exact reference distance: f64, axis order, correctly rounded, no FMA
// (bvh.py:284-290; SURVEY.md hazard H1).
template <int D>
__device__ __forceinline__ double exact_dist(const float* q, const float* p) {
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    double dx = __dsub_rn((double)q[k], (double)p[k]);
    s = __dadd_rn(s, __dmul_rn(dx, dx));
  }
  return __dsqrt_rn(s);
}

// Conservative squared lower bound from q to a box in f32: the per-axis gap
// max(0, lo - q, q - hi) and the sum of squares are all rounded toward -inf,
// so the result never exceeds the exact squared distance (overflow saturates
// at FLT_MAX, still a lower bound).  A leaf is a degenerate box (lo == hi == p),
// for which this is a lower bound on |q - p|^2.
template <int D>
__device__ __forceinline__ float box_lb2(const float* q, const float* lo, const float* hi) {
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    float g = fmaxf(0.f, fmaxf(__fsub_rd(lo[k], q[k]), __fsub_rd(q[k], hi[k])));
    s = __fmaf_rd(g, g, s);
  }
  return s;
}

// f32 pruning threshold that is >= radius^2 for every radius the exact f64
// test could still accept (relative slack 2^-20 covers f64 rounding of w).
__device__ __forceinline__ float prune_r2(double radius) {
  if (!(radius < 1e300)) return __int_as_float(0x7f800000);
  double r2 = radius * radius * (1.0 + 0x1p-20);
  return __double2float_ru(r2);
}

__device__ __forceinline__ double bits_to_radius(unsigned long long b) {
  return b >= 0x7ff0000000000000ull ? __longlong_as_double(0x7ff0000000000000ll) : __longlong_as_double((long long)b);
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

struct Scene {
  double lo[3];
  double inv[3];
  double cellw[3];       // world width of one finest lattice cell per axis (0: zero extent)
  float flo[3];
  float fhi[3];
  long long bad_row;     // first row holding a non-finite coordinate, or LLONG_MAX
  unsigned blocks_done;
  int pad;
};

// Spread the low bits of v so consecutive bits land D positions apart.
__device__ __forceinline__ unsigned long long spread_bits3(unsigned long long v) {
  v &= 0x1fffffull;
  v = (v | (v << 32)) & 0x001f00000000ffffull;
  v = (v | (v << 16)) & 0x001f0000ff0000ffull;
  v = (v | (v << 8)) & 0x100f00f00f00f00full;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}
__device__ __forceinline__ unsigned long long spread_bits2(unsigned long long v) {
  v &= 0x7fffffffull;
  v = (v | (v << 16)) & 0x0000ffff0000ffffull;
  v = (v | (v << 8)) & 0x00ff00ff00ff00ffull;
  v = (v | (v << 4)) & 0x0f0f0f0f0f0f0f0full;
  v = (v | (v << 2)) & 0x3333333333333333ull;
  v = (v | (v << 1)) & 0x5555555555555555ull;
  return v;
}

// Lattice cell of one coordinate (geometry.py:169-177): f64 (x - lo) * inv,
// clamped to [0, nextafter(1, 0)], scaled by 2^bits and truncated.  Monotone
// non-decreasing in x (every step is a correctly rounded monotone operation).
__device__ __forceinline__ unsigned long long lattice_cell_d(double x, double lo, double inv, double scale) {
  double t = __dmul_rn(__dsub_rn(x, lo), inv);
  const double below_one = 0x1.fffffffffffffp-1;
  if (t < 0.0) t = 0.0;
  else if (t > below_one) t = below_one;
  return __double2ull_rz(__dmul_rn(t, scale));
}
__device__ __forceinline__ unsigned long long lattice_cell(float x, double lo, double inv, double scale) {
  return lattice_cell_d((double)x, lo, inv, scale);
}

// Morton code of a lattice cell triple (x most significant), as in k_morton.
template <int D>
__device__ __forceinline__ unsigned long long morton_of_cells(const unsigned long long* c) {
  if (D == 3) return (spread_bits3(c[0]) << 2) | (spread_bits3(c[1]) << 1) | spread_bits3(c[2]);
  return (spread_bits2(c[0]) << 1) | spread_bits2(c[1]);
}

// Length of the Morton prefix shared by every lattice cell the box
// [q - r, q + r] can touch.  The quantiser is monotone per axis, so all points
// inside the box have codes between the codes of its two corners; corners are
// rounded outward and r is inflated past any f64 rounding of a distance, so a
// point whose distance evaluates to <= r cannot fall outside.
template <int D>
__device__ __forceinline__ int ball_prefix(const float* q, double r, const Scene& sc) {
  // Per axis: the high bits shared by the lattice cells of q - r and q + r.  The
  // Morton code of axis k's bit j sits at 64-bit position (64 - D*bits) + D*j + k
  // counted from the top, so the corners' shared code prefix is the minimum of
  // that position over the axes at their first differing bit (no interleaving).
  constexpr int bits = D == 3 ? 21 : 31;
  const double scale = D == 3 ? 2097152.0 : 2147483648.0;
  const double rr = __dmul_ru(r, 1.0 + 0x1p-40);
  int prefix = 64;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const unsigned long long lo = lattice_cell_d(__dsub_rd((double)q[k], rr), sc.lo[k], sc.inv[k], scale);
    const unsigned long long hi = lattice_cell_d(__dadd_ru((double)q[k], rr), sc.lo[k], sc.inv[k], scale);
    const unsigned long long x = lo ^ hi;
    const int pk = (64 - D * bits) + D * (__clzll((long long)x) - (64 - bits)) + k;
    prefix = x ? min(prefix, pk) : prefix;
  }
  return prefix;
}

// Lower bound of the distance from q to any point OUTSIDE the Karras node whose
// Morton prefix has length `pl` (q's own leaf lies under it): such a point's
// code differs from q's within the first pl bits, so on some axis whose bits
// the prefix fixes its lattice cell lies outside q's cell block on that axis.
// The distance to the block's faces loses one finest cell of slack, far more
// than any f64 rounding of the quantiser or of this arithmetic.  pl < 0: the root (no outside).
template <int D>
__device__ __forceinline__ double cell_exterior(const float* q, int pl, const Scene& sc) {
  constexpr int bits = D == 3 ? 21 : 31;
  const double scale = D == 3 ? 2097152.0 : 2147483648.0;
  double best = __longlong_as_double(0x7ff0000000000000ll);
  if (pl < 0) return best;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const int t = pl - (64 - D * bits) - k;   // code positions of axis k inside the prefix: off + D*j + k < pl
    const int bk = t > 0 ? min(bits, (t + D - 1) / D) : 0;
    const double w = sc.cellw[k];   // one finest cell
    if (bk == 0 || !(w > 0.0)) continue;
    const unsigned long long cq = lattice_cell_d((double)q[k], sc.lo[k], sc.inv[k], scale);
    const int sh = bits - bk;
    const unsigned long long c0 = (cq >> sh) << sh, c1 = c0 + (1ull << sh);
    // (offsets from lo, all <= the extent: rounding stays ~1e-15 of the extent,
    // against a slack of one cell, >= 2^-31 of it)
    const double dq = (double)q[k] - sc.lo[k];
    if (c0 > 0) best = fmin(best, dq - (double)c0 * w - w);
    if (c1 < (1ull << bits)) best = fmin(best, (double)c1 * w - dq - w);
  }
  return fmax(best, 0.0);
}

}  // namespace emst
