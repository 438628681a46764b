// traverse.cuh -- the hot kernel: per-query constrained nearest-foreign-neighbour
// search, Algorithm 2 of the paper (reference mst.py:227-328).
//
// B200 design:
//   * persistent warps with lane refill: a lane that finishes its query takes
//     the next one from its warp's chunk of consecutive Morton slots, so warps
//     no longer idle behind their longest query (warp max/mean pops is 1.7-1.9);
//   * one 64-byte node record per pop carries both child boxes, child refs and
//     child component labels (leaf children as degenerate boxes), fetched with
//     four 16-byte loads through the read-only path;
//   * both children get the same branch-free conservative f32 lower bound
//     (rounded toward -inf); only leaves that survive it pay for the exact f64
//     reference distance (bvh.py:284-290) that decides acceptance;
//   * the per-component radius is shared: a query's accepted candidate lowers
//     ub[comp] with a u64 atomicMin on the f64 bit pattern when the query ends,
//     and later queries of the component start from it (long searches also
//     re-read it, kRadiusRefresh).  Any value written is a real outgoing edge of the component, so
//     the radius never drops below the component's minimum -- the result is
//     unchanged ("in the extreme case ...").
//   * per-component result: 128-bit atomic min of (w bits, u << 32 | v).
#pragma once
#include "common.cuh"

// `deep` (the local-memory tail of the traversal stack) is only read below the
// stack top, i.e. after it was written; nvcc cannot see that.
#pragma nv_diag_suppress 549

namespace emst {

#ifdef EMST_VISIT_HIST
// developer instrumentation (EXTRA_NVFLAGS=-DEMST_VISIT_HIST, printed under EMST_TRACE):
// node visits by log2 of the node's slot-range size, climb steps [0] and pops [1]
__device__ unsigned long long g_visit_hist[2][32];
__device__ const int2* g_visit_range;
#endif

template <int D>
__device__ __forceinline__ void child_box(const Node3& rec, int side, float* lo, float* hi) {
  if (side == 0) {
    lo[0] = rec.a.x; lo[1] = rec.a.z; lo[2] = rec.b.x; hi[0] = rec.b.z; hi[1] = rec.c.x; hi[2] = rec.c.z;
  } else {
    lo[0] = rec.a.y; lo[1] = rec.a.w; lo[2] = rec.b.y; hi[0] = rec.b.w; hi[1] = rec.c.y; hi[2] = rec.c.w;
  }
}
template <int D>
__device__ __forceinline__ void child_box(const Node2& rec, int side, float* lo, float* hi) {
  if (side == 0) {
    lo[0] = rec.a.x; lo[1] = rec.a.z; hi[0] = rec.b.x; hi[1] = rec.b.z;
  } else {
    lo[0] = rec.a.y; lo[1] = rec.a.w; hi[0] = rec.b.y; hi[1] = rec.b.w;
  }
  lo[2] = hi[2] = 0.f;
}

// Both children's conservative squared lower bounds at once (box_lb2 for each,
// bit for bit): per axis one packed f32x2 subtraction per face, rounded toward
// -inf, then max(0, .) per child and a packed fma rounded toward -inf.
__device__ __forceinline__ unsigned long long f2pack(float x, float y) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ void f2unpack(unsigned long long r, float& x, float& y) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(r));
}
__device__ __forceinline__ void pair_axis(unsigned long long lo, unsigned long long hi, float qk,
                                          unsigned long long& s) {
  const unsigned long long q2 = f2pack(qk, qk);
  unsigned long long a, b, g;
  asm("sub.rm.f32x2 %0, %1, %2;" : "=l"(a) : "l"(lo), "l"(q2));
  asm("sub.rm.f32x2 %0, %1, %2;" : "=l"(b) : "l"(q2), "l"(hi));
  float a0, a1, b0, b1;
  f2unpack(a, a0, a1);
  f2unpack(b, b0, b1);
  g = f2pack(fmaxf(0.f, fmaxf(a0, b0)), fmaxf(0.f, fmaxf(a1, b1)));
  asm("fma.rm.f32x2 %0, %1, %1, %2;" : "=l"(s) : "l"(g), "l"(s));
}
__device__ __forceinline__ void node_lb2(const Node3& r, const float* q, float& lb0, float& lb1) {
  unsigned long long s = 0ull;   // (+0, +0)
  pair_axis(f2pack(r.a.x, r.a.y), f2pack(r.b.z, r.b.w), q[0], s);
  pair_axis(f2pack(r.a.z, r.a.w), f2pack(r.c.x, r.c.y), q[1], s);
  pair_axis(f2pack(r.b.x, r.b.y), f2pack(r.c.z, r.c.w), q[2], s);
  f2unpack(s, lb0, lb1);
}
__device__ __forceinline__ void node_lb2(const Node2& r, const float* q, float& lb0, float& lb1) {
  unsigned long long s = 0ull;
  pair_axis(f2pack(r.a.x, r.a.y), f2pack(r.b.x, r.b.y), q[0], s);
  pair_axis(f2pack(r.a.z, r.a.w), f2pack(r.b.z, r.b.w), q[1], s);
  f2unpack(s, lb0, lb1);
}

// 256-bit read-only loads (LDG.E.ENL2.256 on sm_100a): a 64-byte Node3 is two
// load instructions instead of four.  Node records are immutable during a launch.
__device__ __forceinline__ void ldg256(const void* p, float4& lo, float4& hi) {
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(lo.x), "=f"(lo.y), "=f"(lo.z), "=f"(lo.w), "=f"(hi.x), "=f"(hi.y), "=f"(hi.z), "=f"(hi.w)
               : "l"(p));
}
__device__ __forceinline__ Node3 load_node(const Node3* p) {
  const float4* f = reinterpret_cast<const float4*>(p);
  Node3 r;
  float4 refs;
  ldg256(f, r.a, r.b);
  ldg256(f + 2, r.c, refs);
  r.ref = make_int4(__float_as_int(refs.x), __float_as_int(refs.y), __float_as_int(refs.z), __float_as_int(refs.w));
  return r;
}
__device__ __forceinline__ Node2 load_node(const Node2* p) {
  const float4* f = reinterpret_cast<const float4*>(p);
  Node2 r;
  r.a = __ldg(f);
  r.b = __ldg(f + 1);
  r.ref = __ldg(reinterpret_cast<const int4*>(f + 2));
  return r;
}

__device__ __forceinline__ unsigned lanemask_lt_u32() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

#ifndef EMST_TRAV_THREADS
#define EMST_TRAV_THREADS 128
#endif
constexpr int kTraverseThreads = EMST_TRAV_THREADS;
// Resident 128-thread blocks per SM.  The 3D proof kernels (rounds >= 3) need
// their registers: 7 blocks = 72 registers, no spill, 28 warps (256-thread
// blocks could only pick 80 registers / 24 warps or 64 with 102 B of spills:
// 37M blobs 3D -1.3 ms for 128 x 7).  Every other variant fits 64 registers
// (8 blocks, 32 warps); 2D lanes prefer the extra warps (-17 % vs 48 warps less).
// Round 1 (kSingle, 8 blocks) and the 3D round-2 kernel (no proof) have their own knobs; the
// round-2 kernel runs 8 blocks at 64 registers (28 B of spills) since its radius refresh is
// clocked by the visit counter: round 2 at 37M blobs 3D 11.58 -> 11.14 ms.
#ifndef EMST_TRAV_MINB3
#define EMST_TRAV_MINB3 7
#endif
#ifndef EMST_TRAV_MINB3S
#define EMST_TRAV_MINB3S 8
#endif
#ifndef EMST_TRAV_MINB3R2
#define EMST_TRAV_MINB3R2 8
#endif
#ifndef EMST_TRAV_MINB2S
#define EMST_TRAV_MINB2S 9
#endif
#ifndef EMST_TRAV_MINB2
#define EMST_TRAV_MINB2 8
#endif
#ifndef EMST_REFILL_IDLE
#define EMST_REFILL_IDLE 16
#endif
#ifndef EMST_REFILL_IDLE3
#define EMST_REFILL_IDLE3 10
#endif
#ifndef EMST_TRAV_CHUNK
#define EMST_TRAV_CHUNK 64
#endif
#ifndef EMST_SMEM_STACK
#define EMST_SMEM_STACK 12
#endif
#ifndef EMST_TRAV_PREFETCH
#define EMST_TRAV_PREFETCH 8192
#endif
#ifndef EMST_TRAV_PF_STAGE
#define EMST_TRAV_PF_STAGE 1
#endif
constexpr long long kTravPrefetch = EMST_TRAV_PREFETCH;   // L2 prefetch lookahead in slots (0: off)
constexpr int kTraverseChunk = EMST_TRAV_CHUNK;   // consecutive Morton queries a warp claims at once
constexpr int kSmemStack = EMST_SMEM_STACK;       // stack entries per lane kept in shared memory
// refill when this many lanes are idle (or all are); measured best: 10 in 3D, 16 in 2D
// (37M blobs 3D traversal 44.58 -> 44.27 ms at 10; 24M blobs 2D +0.4 ms at 10, so 2D keeps 16)
#ifndef EMST_REFILL_IDLE_S
#define EMST_REFILL_IDLE_S 0   // round 1's kernel (0: as the others)
#endif
template <int D, bool kSingle> constexpr int kRefillIdle =
    kSingle && EMST_REFILL_IDLE_S ? EMST_REFILL_IDLE_S : (D == 3 ? EMST_REFILL_IDLE3 : EMST_REFILL_IDLE);
#ifndef EMST_REFRESH_BY_VISITS
#define EMST_REFRESH_BY_VISITS 1
#endif
#ifndef EMST_DONE_PREFETCH
#define EMST_DONE_PREFETCH 0   // L1 prefetch of the candidate point when a query ends (measured: off is 0.1-0.5 ms faster)
#endif
#ifndef EMST_STACK_FAST
#define EMST_STACK_FAST 1   // pushes branch once on "all in shared memory" (1); pops and single pushes too (2)
#endif
#ifndef EMST_RADIUS_REFRESH
#define EMST_RADIUS_REFRESH 4096
#endif
// visits between re-reads of the component's shared radius (the lane's visit
// counter is the clock).  Measured at 37M blobs 3D: every 16 pops 72.4 ms, 32:
// 71.8, 64: 71.4, 256: 70.6 (round 1); round 2, traversal 43.8 ms at 256, 43.6 at
// 512, 43.5 at 1024, 43.4 at 4096 and 43.3 at 65536 -- an L2 read per lane costs
// more than the slightly tighter radius saves; only very long searches re-read.
constexpr int kRadiusRefresh = EMST_RADIUS_REFRESH;
#ifndef EMST_SHARE_AT_END
#define EMST_SHARE_AT_END 1
#endif
// publish a query's candidate to the component bound when it ends (batched with
// the other finished lanes) instead of on every improvement
constexpr bool kShareAtEnd = EMST_SHARE_AT_END;      // pops between re-reads of the shared radius

// f32 upper bound of |q - p|^2 (every operation rounded toward +inf).
template <int D>
__device__ __forceinline__ float point_ub2(const float* q, const float* p) {
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const float g = fmaxf(__fsub_ru(q[k], p[k]), __fsub_ru(p[k], q[k]));
    s = __fmaf_ru(g, g, s);
  }
  return s;
}

// Exact reference key (w bits, u << 32 | v) of the edge from query (q, qp) to
// the point in slot `slot` (mst.py:270-289; bvh.py:284-290).  With core
// distances (mutual reachability, slot order) the weight is
// max(d, core(p), core(q)) (mst.py:278-281).
template <int D>
__device__ __forceinline__ void exact_key(const float* q, unsigned qp, const float4* __restrict__ spts, int slot,
                                          unsigned long long& w, unsigned long long& uv,
                                          const double* __restrict__ core = nullptr, double cq = 0.0) {
  const float4 pv = __ldg(spts + slot);
  const float p[3] = {pv.x, pv.y, pv.z};
  double wd = exact_dist<D>(q, p);
  if (core) wd = fmax(wd, fmax(__ldg(core + slot), cq));
  w = (unsigned long long)__double_as_longlong(wd);
  const unsigned pp = __float_as_uint(pv.w);
  const unsigned long long u = qp < pp ? qp : pp, v = qp < pp ? pp : qp;
  uv = (u << 32) | v;
}

// A query's best foreign leaf so far, kept as its slot and an f32 interval
// [lo, hi] around the squared distance.  The exact f64 weight (the only value
// that decides acceptance and order) is evaluated once, when the query ends,
// for all finished lanes of the warp together; the interval alone decides
// almost every comparison on the way, because two candidates whose intervals
// are disjoint are separated by >= 1 f32 ulp of d^2 and their f64 weights
// (error ~2^-52) order the same way.  Overlapping intervals (near-ties) are
// resolved exactly on the spot.
struct Pending {
  int slot;   // -1: none
  float lo, hi;
};

// Visit one child of a fetched node record: the f32 lower bound, the component
// skip (leaves always, mst.py:276; subtrees under subtree_skip, mst.py:291) and,
// for a surviving leaf, the candidate update.  Pruning stays conservative: r2
// never drops below the squared distance of a real foreign candidate, and a
// box is pruned only when its lower bound is strictly above r2 (ties at the
// radius are kept, mst.py:259/282/296).  Returns true when an internal child
// should be explored (lb in *lb_out).
template <int D, bool kSkip, bool kBounds, bool kProof, bool kSingle, class Rec>
__device__ __forceinline__ bool visit_child(const Rec& rec, int side, const float* q, unsigned qp, int comp,
                                            float& r2, Pending& pend, const float4* __restrict__ spts,
                                            unsigned long long* ub, bool share, unsigned& evals, float lb,
                                            bool enabled, const double* __restrict__ core, double cq,
                                            float& pmin2) {
  const int c = side ? rec.ref.y : rec.ref.x;
  const int cl = side ? rec.ref.w : rec.ref.z;
  // (round 1: every point is its own component and the query never visits its own leaf)
  const bool same = !kSingle && cl == comp && (c < 0 || kSkip);
  if (!enabled || same || lb > r2) return false;
  if (c >= 0) return true;
  ++evals;
  float lo[3], hi[3];
  child_box<D>(rec, side, lo, hi);
  float ub2 = point_ub2<D>(q, lo);
  if (core) {
    // mutual reachability: the weight's square lies in [max(lb, cm^2), max(ub2, cm^2)]
    const double cm = fmax(__ldg(core + ~c), cq);
    lb = fmaxf(lb, __double2float_rd(__dmul_rd(cm, cm)));
    ub2 = fmaxf(ub2, __double2float_ru(__dmul_ru(cm, cm)));
    if (lb > r2) return false;
  }
  if (pend.slot < 0 || ub2 < pend.lo) {
    pend.slot = ~c;   // strictly nearer than the pending candidate (or the first)
    pend.lo = lb;
    pend.hi = ub2;
  } else if (!(lb > pend.hi)) {
    // overlapping intervals: compare the exact keys
    unsigned long long wa, uva, wb, uvb;
    exact_key<D>(q, qp, spts, pend.slot, wa, uva, core, cq);
    exact_key<D>(q, qp, spts, ~c, wb, uvb, core, cq);
    if (key_less(wb, uvb, wa, uva)) {
      pend.slot = ~c;
      pend.lo = lb;
      pend.hi = ub2;
    }
  } else {
    return false;   // strictly farther than the pending candidate
  }
  if (pend.hi < r2) {
    r2 = pend.hi;
    // Share it with the component's other queries: an upper bound of the
    // candidate's weight (sqrt rounded up, then 2^-40 slack over any f64
    // rounding of the exact weight) is at least the weight of a real outgoing
    // edge, so it is a valid radius for every query of the component.
    if (kBounds && share && !kShareAtEnd)
      atomicMin(&ub[comp], (unsigned long long)__double_as_longlong(__dmul_ru((double)__fsqrt_ru(pend.hi), 1.0 + 0x1p-40)));
  }
  return false;
}

// Bottom-up ("climb") traversal.  A query starts at its own leaf and climbs the
// Karras tree; at every ancestor it explores only the sibling subtree (top-down,
// nearest first, with the stack), so the root-to-leaf path is never walked
// downward.  The climb stops at the first ancestor whose Morton prefix is no
// longer than the prefix shared by the query's whole search box [q - r, q + r]:
// every point within r has a code with that prefix, and a Karras node holds ALL
// points with its prefix, so nothing outside that ancestor can be within r.
// In round 1 (radius = distance to a Z-order neighbour) this stops a few levels
// above the leaf instead of walking ~38 levels down from the root.
//
// Stack: the first kSmemStack entries of every lane live in shared memory laid
// out [depth][thread] (bank = lane for every depth, so lanes at different depths
// never conflict); deeper entries, rare, spill to a per-thread local array up to
// the reference's capacity of 64 (bvh.py:36).
// kProof: record the search's full nearest-foreign proof (pruned lower bounds
// and the stop node's cell, see cell_exterior) instead of just the radius; it
// lets later rounds settle more queries up front, and costs a little per visit.
// kSingle: round 1 compiled on its own (every query its own component, nothing
// is ever "same component", no shared radius).
template <int D, bool kSkip, bool kBounds, bool kMrd, bool kProof, bool kSingle>
__global__ void __launch_bounds__(kTraverseThreads, D == 3 ? (kSingle ? EMST_TRAV_MINB3S : kProof ? EMST_TRAV_MINB3 : EMST_TRAV_MINB3R2) : (kSingle ? EMST_TRAV_MINB2S : EMST_TRAV_MINB2))
k_traverse(const typename NodeOf<D>::type* __restrict__ nodes, const float4* __restrict__ spts,
           const unsigned* __restrict__ perm, const int* __restrict__ label, unsigned long long* ub,
           EdgeKey* __restrict__ best, long long q0, long long q1, const Box3* __restrict__ root_box,
           unsigned long long* __restrict__ evals_out, int* __restrict__ overflow,
           unsigned long long* __restrict__ work_counter, bool singletons, float* __restrict__ nfn_lb,
           const int2* __restrict__ up, const int* __restrict__ leaf_parent, const Scene* __restrict__ scene_ptr,
           const int* __restrict__ top_pure_in, const double* __restrict__ core_in, const int* __restrict__ side_in,
           const int* __restrict__ qlist_in, const unsigned* __restrict__ qcount, int claim) {
  // round 1 (kSingle) has no pure nodes, no one-sided round, no query list and no earlier proofs
  const int* __restrict__ top_pure = kSingle ? nullptr : top_pure_in;
  // (query lists and the one-sided last round come with the proof kernels only)
  const int* __restrict__ side = kSingle || !kProof ? nullptr : side_in;
  const int* __restrict__ qlist = kSingle || !kProof ? nullptr : qlist_in;
  constexpr bool kNlb = kBounds && !kSingle;
  // qlist: the slots to run (k_prefilter dropped the ones settled up front), else all of [q0, q1)
  // mutual reachability (kMrd): core distances per slot; compiled out otherwise
  const double* __restrict__ core = kMrd ? core_in : nullptr;
  const unsigned lane = lane_id();
  const unsigned lt = lanemask_lt_u32();
  const int total = qlist ? (int)*qcount : (int)(q1 - q0);
  const Scene sc = *scene_ptr;
  const int skip_comp = side ? *side : -1;   // last round: the component whose queries are not run

  // The warp claims `claim` (<= kTraverseChunk) consecutive Morton slots at a time and stages
  // their point, label, leaf parent, starting radius, proven nearest-foreign
  // bound and top pure node in shared memory with coalesced loads.
  constexpr int W = kTraverseThreads / 32;
  __shared__ float4 s_pts[W][kTraverseChunk];
  __shared__ int s_lab[W][kTraverseChunk];
  __shared__ int s_lp[W][kTraverseChunk];
  __shared__ unsigned long long s_ub[W][kTraverseChunk];
  __shared__ float s_nlb[W][kTraverseChunk];
  __shared__ int s_top[W][kTraverseChunk];
  __shared__ int s_slot[W][kTraverseChunk];
  __shared__ int2 s_stk[kSmemStack][kTraverseThreads];
  int2 deep[kStackCapacity - kSmemStack];
  const int wib = threadIdx.x >> 5;
  const int tid = threadIdx.x;
  int chunk_base = 0;
  int pool_next = 0, pool_end = 0;   // warp-uniform chunk of claimed queries
  bool exhausted = false;            // warp-uniform: global work is gone

  int s = -1;
  float q[3] = {0.f, 0.f, 0.f};
  unsigned qp = 0;
  int comp = 0;
  double radius = 0.0;
  float r2 = 0.f;
  float my_nlb = 0.f;
  double cq = 0.0;   // core distance of the query (mutual reachability)
  Pending pend{-1, 0.f, 0.f};
  int top = 0;
  int climb = -1;          // ancestor whose sibling subtree is next, -1 = climb over
  int path_side = 0;       // which child of `climb` the query came from
  int prefix = 0;          // Morton prefix shared by the search box
  float prefix_r2 = 0.f;   // r2 `prefix` was computed for
  int since_refresh = 0;
  // nearest-foreign proof of the search: the smallest lower bound of anything it
  // pruned, and the prefix length of the node its climb stopped at (everything
  // outside that node is at least cell_exterior away); -1: the climb reached the
  // root, -2: the query was settled without a search
  float pmin2 = 0.f;
  int stop_pl = -2;
  unsigned evals = 0, visits = 0, found = 0, skipped = 0;
  // A finished query keeps its state until the warp refills: the exact weight
  // of its candidate, the nearest-foreign bound and the 128-bit atomic min then
  // run for all finished lanes together instead of one divergent lane at a time.
  bool done = false;

  auto finalize = [&]() {
    unsigned long long w = ~0ull, uv = ~0ull;
    double proven = radius;
    if (kProof && stop_pl != -2)
      proven = fmin(cell_exterior<D>(q, stop_pl, sc), (double)__fsqrt_rd(pmin2));
    if (pend.slot >= 0) {
      exact_key<D>(q, qp, spts, pend.slot, w, uv, core, cq);
      const double wd = __longlong_as_double((long long)w);
      if (wd < proven) proven = wd;
      // (a strictly smaller radius means another query already beat this edge)
      if (!(wd > radius)) {
        ++found;
        if (kSingle || singletons) {
          store_key(&best[comp], w, uv);   // round 1: the query is its component
        } else {
          if (kBounds && kShareAtEnd && w < __ldcg(&ub[comp])) atomicMin(&ub[comp], w);
          atomic_min_key(&best[comp], w, uv);
        }
      }
    }
    // the search proved: no foreign point closer than `proven` (a Euclidean
    // statement: with core distances the search bounds weights, not distances)
    if (kBounds && !core) {
      const float pr = __double2float_rd(__dmul_rd(proven, 1.0 - 0x1p-40));
      if (pr > my_nlb) nfn_lb[s] = pr;
    }
    done = false;
    s = -1;
  };

  // entry i of this lane's stack is at stk0 + i * kStkStride in the shared window
  // (kept opaque so that the compiler holds it in one register instead of
  // re-deriving it from %tid / %cgactaid at every stack access)
  unsigned stk0;
  asm volatile("mov.u32 %0, %1;" : "=r"(stk0) : "r"((unsigned)__cvta_generic_to_shared(&s_stk[0][tid])));
  constexpr unsigned kStkStride = kTraverseThreads * sizeof(int2);
  auto stk_get = [&](int i) -> int2 {
    if (i < kSmemStack) {
      int2 e;
      asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(e.x), "=r"(e.y) : "r"(stk0 + i * kStkStride));
      return e;
    }
    return deep[i - kSmemStack];
  };
  auto stk_put = [&](int i, int node, float lb) {
    if (i < kSmemStack)
      asm volatile("st.shared.v2.s32 [%0], {%1, %2};" :: "r"(stk0 + i * kStkStride), "r"(node), "r"(__float_as_int(lb)) : "memory");
    else
      deep[i - kSmemStack] = make_int2(node, __float_as_int(lb));
  };

  for (;;) {
    // ---- refill idle lanes from the warp's staged chunk of consecutive Morton slots
    const unsigned idle = __ballot_sync(0xffffffffu, s < 0 || done);
    const int n_idle = __popc(idle);
    if (n_idle == 32 && exhausted) {
      if (done) finalize();
      break;
    }
    if (n_idle >= kRefillIdle<D, kSingle>) {   // warp-uniform
      if (done) finalize();
      if (pool_next >= pool_end && !exhausted) {
        unsigned long long base = 0;
        if (lane == 0) {
          base = atomicAdd(work_counter, (unsigned long long)claim);
#if EMST_TRAV_PREFETCH
          // Warm L2 for the queries kTravPrefetch slots ahead: the low tree levels
          // they start in are the node records of about the same indices (Karras
          // numbering), and first touches of those are the traversal's DRAM reads.
          // (not for listed queries: warming the slots around the listed ones measured neutral)
          const long long a = q0 + (long long)base + kTravPrefetch;
          if (!qlist && a + kTraverseChunk < q1) {
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;"
                         :: "l"(nodes + a), "r"((unsigned)(kTraverseChunk * sizeof(*nodes))) : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;"
                         :: "l"(spts + a), "r"((unsigned)(kTraverseChunk * sizeof(float4))) : "memory");
#if EMST_TRAV_PF_STAGE
            // the per-slot words the chunk staging loads (4-byte arrays: 16-byte aligned when a is a multiple of 4)
            if ((a & 3) == 0) {
              const unsigned bytes = (unsigned)(kTraverseChunk * sizeof(int));
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(label + a), "r"(bytes) : "memory");
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(leaf_parent + a), "r"(bytes) : "memory");
              if (kNlb) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(nfn_lb + a), "r"(bytes) : "memory");
              if (top_pure) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(top_pure + a), "r"(bytes) : "memory");
            }
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;"
                         :: "l"(up + a), "r"((unsigned)(kTraverseChunk * sizeof(int2))) : "memory");
#endif
          }
#endif
        }
        base = __shfl_sync(0xffffffffu, base, 0);
        if ((long long)base >= total) {
          exhausted = true;
        } else {
          chunk_base = (int)base;
          pool_next = chunk_base;
          pool_end = min(chunk_base + claim, total);
          __syncwarp();
#pragma unroll
          for (int j = 0; j < kTraverseChunk / 32; ++j) {
            const int i = chunk_base + j * 32 + (int)lane;
            if (i < pool_end) {
              const long long g = qlist ? (long long)qlist[i] : q0 + i;
              if (qlist) s_slot[wib][j * 32 + lane] = (int)g;
              s_pts[wib][j * 32 + lane] = spts[g];
              s_lab[wib][j * 32 + lane] = label[g];
              s_lp[wib][j * 32 + lane] = leaf_parent[g];
              if (kNlb) s_nlb[wib][j * 32 + lane] = nfn_lb[g];
              if (top_pure) s_top[wib][j * 32 + lane] = top_pure[g];
            }
          }
          if (kBounds) {
            __syncwarp();
#pragma unroll
            for (int j = 0; j < kTraverseChunk / 32; ++j) {
              const int i = chunk_base + j * 32 + (int)lane;
              if (i < pool_end) s_ub[wib][j * 32 + lane] = __ldcg(&ub[s_lab[wib][j * 32 + lane]]);
            }
          }
          __syncwarp();
        }
      }
      if (pool_next < pool_end) {
        const int rank = __popc(idle & lt);
        const int mine = pool_next + rank;
        const bool take = s < 0 && mine < pool_end;
        pool_next = min(pool_end, pool_next + n_idle);
        if (take) {
          const int k = mine - chunk_base;
          s = qlist ? s_slot[wib][k] : (int)(q0 + mine);   // the query's slot
          const float4 qv = s_pts[wib][k];
          q[0] = qv.x; q[1] = qv.y; q[2] = qv.z;
          qp = __float_as_uint(qv.w);
          comp = s_lab[wib][k];
          radius = kBounds ? bits_to_radius(s_ub[wib][k]) : __longlong_as_double(0x7ff0000000000000ll);
          r2 = prune_r2(radius);
          pend.slot = -1;
          top = 0;
          const int link = s_lp[wib][k];
          climb = link >> 1;
          path_side = link & 1;
          prefix = radius < 1e300 ? ball_prefix<D>(q, radius, sc) : -1;
          prefix_r2 = r2;
          since_refresh = kRadiusRefresh / 2;   // staged radius may be stale: refresh early
          pmin2 = __int_as_float(0x7f800000);
          my_nlb = kNlb ? s_nlb[wib][k] : 0.f;
          // A previous round proved every foreign point is farther than nfn_lb[s]
          // (foreign sets only shrink, so that stays true).  If that already
          // exceeds the radius, this query cannot find an edge: done.
          if (kNlb && (double)my_nlb > radius) climb = -1;
          // last round: the other component's queries find the same edge
          if (comp == skip_comp) climb = -1;
          // mutual reachability: every edge of q weighs at least core(q)
          if (core) {
            cq = __ldg(core + s);
            if (cq > radius) climb = -1;
          }
          // Every leaf under the query's top pure node T is in its own component:
          // the climb starts above T, and if the search box's prefix already lies
          // inside T there is nothing foreign within the radius at all.
          if (top_pure && climb >= 0) {
            const int t = s_top[wib][k];
            if (t > 0) {
              const int2 ut = __ldg(up + (t - 1));
              if (ut.y <= prefix || ut.x < 0) {
                climb = -1;
              } else {
                climb = ut.x >> 1;
                path_side = ut.x & 1;
              }
            }
          }
          skipped += climb < 0;
          stop_pl = climb < 0 ? -2 : -1;
        }
      }
    }
    if (s < 0 || done) continue;

#if EMST_RADIUS_REFRESH == 0
    if (false) {   // (no refresh: the staged radius stands for the whole search)
#elif EMST_REFRESH_BY_VISITS
    // (the lane's visit counter doubles as the refresh clock: one increment per step less)
    if (kBounds && !(kSingle || singletons) && (visits & (kRadiusRefresh - 1)) == kRadiusRefresh - 1) {
#else
    if (kBounds && !(kSingle || singletons) && ++since_refresh >= kRadiusRefresh) {
      since_refresh = 0;
#endif
      const double shared = bits_to_radius(__ldcg(&ub[comp]));
      if (shared < radius) { radius = shared; r2 = fminf(r2, prune_r2(shared)); }
    }
    // ---- one node visit per iteration, the same code for both kinds of step so
    // that lanes popping a parked subtree and lanes climbing do not diverge:
    //   pop:   both children of a parked node (top-down, nearest first)
    //   climb: only the sibling of the path under ancestor `climb`
    // Parked entries the radius has since pruned are dropped first.
    int2 e = make_int2(-1, 0);
    while (top > 0) {
#if EMST_STACK_FAST >= 2
      if (top <= kSmemStack)
        asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(e.x), "=r"(e.y) : "r"(stk0 + (top - 1) * kStkStride));
      else
        e = deep[top - 1 - kSmemStack];
#else
      e = stk_get(top - 1);
#endif
      if (__int_as_float(e.y) <= r2) break;
      if (kProof) pmin2 = fminf(pmin2, __int_as_float(e.y));
      --top;
      e.x = -1;
    }
    const bool climbing = top == 0;
    // pop: both children; climb: only the sibling of the path (climb is -1 when the climb is over).
    // (plain selects and two booleans: the unsigned side mask of the earlier form was rebuilt by
    // the compiler at each use, ~8 instructions per step -- 37M blobs 3D 66.3 -> 65.6 ms)
    const int node = climbing ? climb : e.x;
    top -= !climbing;
    const bool en0 = !climbing || path_side != 0, en1 = !climbing || path_side == 0;
    if (node >= 0) {
      ++visits;
#ifdef EMST_VISIT_HIST
      {
        const int2 rg = g_visit_range[node];
        atomicAdd(&g_visit_hist[climbing ? 0 : 1][31 - __clz(rg.y - rg.x + 1)], 1ull);
      }
#endif
      const auto rec = load_node(nodes + node);
      int2 u = make_int2(-1, 0);
      if (climbing) u = __ldg(up + node);   // (parent link, prefix length of `climb`)
      float lb0, lb1;
      node_lb2(rec, q, lb0, lb1);
      const bool w0 = visit_child<D, kSkip, kBounds, kProof, kSingle>(rec, 0, q, qp, comp, r2, pend, spts, ub, !(kSingle || singletons), evals,
                                                     lb0, en0, core, cq, pmin2);
      const bool w1 = visit_child<D, kSkip, kBounds, kProof, kSingle>(rec, 1, q, qp, comp, r2, pend, spts, ub, !(kSingle || singletons), evals,
                                                     lb1, en1, core, cq, pmin2);
      const bool want0 = w0 && lb0 <= r2, want1 = w1 && lb1 <= r2;
      // (a child the other one's candidate has since put beyond r2 is pruned too)
      if (kProof) {
        // every foreign (or mixed) child not pushed, pruned or a leaf already
        // tested: nothing in it is nearer than its lower bound
        const bool f0 = en0 && !want0 && !(rec.ref.z == comp && (rec.ref.x < 0 || kSkip));
        const bool f1 = en1 && !want1 && !(rec.ref.w == comp && (rec.ref.y < 0 || kSkip));
        pmin2 = fminf(pmin2, fminf(f0 ? lb0 : __int_as_float(0x7f800000), f1 ? lb1 : __int_as_float(0x7f800000)));
      }
      const int np = (int)want0 + (int)want1;
      if (top + np > kStackCapacity) {
        atomicOr(overflow, 1);
        top = 0;
        climb = -1;
        stop_pl = -2;
      } else if (np == 2) {
        // nearer child on top (popped first); ties keep the left child there
        const bool near1 = lb1 < lb0;
#if EMST_STACK_FAST
        if (top + 2 <= kSmemStack) {   // (the common case: both entries in shared memory, one branch)
          asm volatile("st.shared.v2.s32 [%0], {%1, %2};" :: "r"(stk0 + top * kStkStride),
                       "r"(near1 ? rec.ref.x : rec.ref.y), "r"(__float_as_int(near1 ? lb0 : lb1)) : "memory");
          asm volatile("st.shared.v2.s32 [%0], {%1, %2};" :: "r"(stk0 + (top + 1) * kStkStride),
                       "r"(near1 ? rec.ref.y : rec.ref.x), "r"(__float_as_int(near1 ? lb1 : lb0)) : "memory");
        } else {
          stk_put(top, near1 ? rec.ref.x : rec.ref.y, near1 ? lb0 : lb1);
          stk_put(top + 1, near1 ? rec.ref.y : rec.ref.x, near1 ? lb1 : lb0);
        }
#else
        stk_put(top, near1 ? rec.ref.x : rec.ref.y, near1 ? lb0 : lb1);
        stk_put(top + 1, near1 ? rec.ref.y : rec.ref.x, near1 ? lb1 : lb0);
#endif
        top += 2;
      } else if (np == 1) {
#if EMST_STACK_FAST >= 2
        if (top < kSmemStack)
          asm volatile("st.shared.v2.s32 [%0], {%1, %2};" :: "r"(stk0 + top * kStkStride),
                       "r"(want0 ? rec.ref.x : rec.ref.y), "r"(__float_as_int(want0 ? lb0 : lb1)) : "memory");
        else
#endif
        stk_put(top, want0 ? rec.ref.x : rec.ref.y, want0 ? lb0 : lb1);
        ++top;
      }
      if (climbing && climb >= 0) {
        // Only points with d^2 <= r2 can still matter (anything farther is
        // beyond the radius or strictly behind the pending candidate).  A prefix
        // computed for a larger r2 is still valid (earlier stopping is never
        // required); refresh it when the climb would go on and the search radius
        // has at least halved since.
        if (u.y > prefix && r2 <= 0.25f * prefix_r2) {
          prefix = ball_prefix<D>(q, (double)__fsqrt_ru(r2), sc);
          prefix_r2 = r2;
        }
        if (u.y <= prefix || u.x < 0) {
          stop_pl = u.x < 0 ? -1 : u.y;
          climb = -1;   // every point within the radius lies under this ancestor
        } else {
          climb = u.x >> 1;
          path_side = u.x & 1;
        }
      }
    }
    if (top == 0 && climb < 0) {
      done = true;
      // finalize() reads the candidate's point at the next refill: start the
      // fetch now so that it is an L1 hit by then
#if EMST_DONE_PREFETCH
      if (pend.slot >= 0) asm volatile("prefetch.global.L1 [%0];" :: "l"(spts + pend.slot));
#endif
    }
  }
  unsigned long long ev64 = evals, vi64 = visits, fo64 = found, sk64 = skipped;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ev64 += __shfl_xor_sync(0xffffffffu, ev64, o);
    vi64 += __shfl_xor_sync(0xffffffffu, vi64, o);
    fo64 += __shfl_xor_sync(0xffffffffu, fo64, o);
    sk64 += __shfl_xor_sync(0xffffffffu, sk64, o);
  }
  if (lane == 0) {
    if (ev64) atomicAdd(evals_out, ev64);
    if (vi64) atomicAdd(evals_out + 5, vi64);   // counters[5]: node visits
    if (fo64) atomicAdd(evals_out + 6, fo64);   // counters[6]: queries with a candidate
    if (sk64) atomicAdd(evals_out + 9, sk64);   // counters[9]: queries settled before any visit
  }
}

}  // namespace emst
