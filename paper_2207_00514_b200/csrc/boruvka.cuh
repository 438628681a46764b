// boruvka.cuh -- per-round kernels of the single-tree Boruvka loop (mst.py:680-732).
//
// State lives in slot space with dense component ids: label[s] in [0, c) for
// the c live components of the round.  Per-component arrays are c-sized, so
// they shrink ~3.4x per round and become L2-resident after round two.
//
//   k_round_scan    one pass over labels: Z-adjacent pairs in different
//                   components seed both upper bounds with their exact f64
//                   weight (u64 atomicMin on the bit pattern; order-independent,
//                   so equal to the serial fold of mst.py:198-224), and the
//                   boundary flags are prefix-summed into B[s]
//   k_node_labels   a node's child label is uniform iff no boundary falls in
//                   the child's slot range: B[hi] == B[lo] (mst.py:185-195)
//   k_traverse      Algorithm 2 (mst.py:227-328): one thread per Morton-ordered
//                   query, short stack, conservative f32 box pruning, exact f64
//                   leaf weights, 128-bit atomic min per component (w, u, v)
//   k_merge_*       successor, chain collapse by pointer jumping, edge emission
//                   and new dense ids (mst.py:351-433)
#pragma once
#include "common.cuh"
#include "scan.cuh"
#include "traverse.cuh"

namespace emst {

// ---------------------------------------------------------------- bounds + B
// One scan over the labels: the boundary flags label[i] != label[i+1] are
// prefix-summed into B[i] (exclusive), and with bounds on, each boundary pair
// seeds both components' upper bounds with its exact f64 weight (u64 min of
// the bit pattern; order-independent, so equal to the serial fold of
// mst.py:198-224).  The 8 items of a thread issue their point loads together,
// then their bound reads, and only the pairs that can still lower a bound
// send an atomic (late rounds funnel many boundaries into few components).
// Lower ub[l] to w for the (l, w) pairs of every lane (l < 0: none).  Dense
// warps (early rounds: distinct labels) read each bound and send an atomic
// only where it can still lower it.  Sparse warps (late rounds: few
// components, many boundaries per component) first reduce per label across
// the warp, so a component receives one atomic per warp instead of one per
// boundary.
template <int K>
__device__ __forceinline__ void apply_bound_updates(int* ul, unsigned long long* uw, unsigned long long* ub) {
  unsigned pending = 0;
#pragma unroll
  for (int j = 0; j < K; ++j) pending |= ul[j] >= 0 ? 1u << j : 0u;
  const unsigned busy = __ballot_sync(0xffffffffu, pending != 0);
  if (__popc(busy) > 8) {
    unsigned long long cur[K];
#pragma unroll
    for (int j = 0; j < K; ++j) cur[j] = ul[j] >= 0 ? __ldcg(&ub[ul[j]]) : 0ull;
#pragma unroll
    for (int j = 0; j < K; ++j)
      if (uw[j] < cur[j]) atomicMin(&ub[ul[j]], uw[j]);
    return;
  }
  const unsigned lane = lane_id();
  for (;;) {
    const unsigned has = __ballot_sync(0xffffffffu, pending != 0);
    if (!has) break;
    const int leader = __ffs(has) - 1;
    const int first = pending ? __ffs(pending) - 1 : 0;
    int mine_l = -1;
#pragma unroll
    for (int j = 0; j < K; ++j) if (j == first) mine_l = ul[j];
    const int L = __shfl_sync(0xffffffffu, mine_l, leader);
    unsigned long long w = ~0ull;
#pragma unroll
    for (int j = 0; j < K; ++j)
      if ((pending >> j & 1u) && ul[j] == L) { w = min(w, uw[j]); pending &= ~(1u << j); }
    const unsigned hi = __reduce_min_sync(0xffffffffu, (unsigned)(w >> 32));
    const unsigned lo = __reduce_min_sync(0xffffffffu, (unsigned)(w >> 32) == hi ? (unsigned)w : 0xffffffffu);
    if ((int)lane == leader) {
      const unsigned long long m = ((unsigned long long)hi << 32) | lo;
      if (m < __ldcg(&ub[L])) atomicMin(&ub[L], m);
    }
  }
}

// A boundary pair's contribution to a component bound.  The building block
// compute_upper_bounds returns the reference's exact f64 weights (mst.py:198-224);
// inside the solve a bound only has to be at least a real edge's weight (H3), so
// an f32 upper bound (every operation rounded up, then 2^-40 of slack over the
// f64 rounding of the exact weight) replaces the f64 distance and its sqrt.
template <int D>
__device__ __forceinline__ unsigned long long seed_weight(const float* pa, const float* pb, bool exact) {
  if (exact) return (unsigned long long)__double_as_longlong(exact_dist<D>(pa, pb));
  return (unsigned long long)__double_as_longlong(__dmul_ru((double)__fsqrt_ru(point_ub2<D>(pa, pb)), 1.0 + 0x1p-40));
}

struct RoundScanOp {
  using T = unsigned;
  static constexpr bool kCached = false;
  static constexpr bool kWarpStore = false;
  const int* label;
  const float4* spts;
  unsigned long long* ub;
  int* bprefix;
  long long n;
  int dim;
  bool bounds;
  const double* core;   // mutual reachability (slot order), or nullptr
  bool exact;           // exact f64 weights (the building block) or upper bounds (the solve)
  // the boundary pairs (s, s + 1) seeded: left slot s in [seed0, seed1) -- a rank of a
  // multi-GPU solve seeds its own Morton range (the ranges tile [0, n - 1), so the
  // min-allreduce of the bounds that follows gives every rank the replicated result)
  long long seed0, seed1;
  __device__ void load(long long i0, int cnt, unsigned* v) const {
    int lab[kScanItems + 1];
#pragma unroll
    for (int j = 0; j <= kScanItems; ++j) lab[j] = 0;
    load8(label, i0, cnt, lab);
    if (i0 + kScanItems < n) lab[kScanItems] = __ldg(label + i0 + kScanItems);
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) v[j] = (i0 + j + 1 < n && lab[j] != lab[j + 1]) ? 1u : 0u;
  }
  // the bound seeding runs after the tile's prefix is out
  __device__ void side(long long i0, int cnt, const unsigned* v) const {
    if (!bounds) return;   // (warp-uniform)
    int lab[kScanItems + 1];
#pragma unroll
    for (int j = 0; j <= kScanItems; ++j) lab[j] = 0;
    load8(label, i0, cnt, lab);
    if (i0 + kScanItems < n) lab[kScanItems] = __ldg(label + i0 + kScanItems);
    unsigned long long wb[kScanItems];
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
      wb[j] = ~0ull;
      if (v[j] && i0 + j >= seed0 && i0 + j < seed1) {
        const float4 a = __ldg(spts + i0 + j), b = __ldg(spts + i0 + j + 1);
        const float pa[3] = {a.x, a.y, a.z}, pb[3] = {b.x, b.y, b.z};
        wb[j] = dim == 3 ? seed_weight<3>(pa, pb, exact) : seed_weight<2>(pa, pb, exact);
        if (core)   // mst.py:217-220
          wb[j] = (unsigned long long)__double_as_longlong(
              fmax(__longlong_as_double((long long)wb[j]), fmax(core[i0 + j], core[i0 + j + 1])));
      }
    }
    // One update per run of equal labels among the thread's 9 slots: the min of
    // the (at most two) boundary weights around the run.
    int ul[kScanItems + 1];
    unsigned long long uw[kScanItems + 1];
    // (slot kScanItems is the next thread's first; it exists iff i0 + 8 < n)
    const int last = i0 + kScanItems < n ? kScanItems : cnt - 1;
    unsigned long long run = ~0ull;
#pragma unroll
    for (int j = 0; j <= kScanItems; ++j) {
      if (j > 0 && v[j - 1]) run = min(run, wb[j - 1]);          // boundary left of slot j
      if (j < kScanItems && v[j]) run = min(run, wb[j]);         // boundary right of slot j
      const bool run_ends = j == last || (j < kScanItems && v[j]);
      ul[j] = j <= last && run_ends && run != ~0ull ? lab[j] : -1;
      uw[j] = run;
      if (run_ends) run = ~0ull;
    }
    apply_bound_updates<kScanItems + 1>(ul, uw, ub);   // every lane of the warp takes part
  }
  __device__ void store(long long i0, int cnt, const unsigned* v, unsigned ex) const {
    int out[kScanItems];
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
      out[j] = (int)ex;
      ex += v[j];
    }
    store8(bprefix, i0, cnt, out);
  }
};

// Round 1 with a wider Z-window: ub[s] = the smallest upper bound of |s - t| over
// the slots t within +-W of s (singletons: no labels, no atomics).  The points of
// a block and its halo are staged in shared memory.
constexpr int kSeed1Threads = 256;
template <int D, int W>
__global__ void __launch_bounds__(kSeed1Threads) k_seed_round1_window(const float4* __restrict__ spts, long long n,
                                                                      unsigned long long* __restrict__ ub) {
  __shared__ float4 sp[kSeed1Threads + 2 * W];
  const long long base = blockIdx.x * (long long)kSeed1Threads;
  for (int i = threadIdx.x; i < kSeed1Threads + 2 * W; i += kSeed1Threads) {
    const long long g = base - W + i;
    sp[i] = g >= 0 && g < n ? spts[g] : make_float4(__int_as_float(0x7f800000), 0.f, 0.f, 0.f);
  }
  __syncthreads();
  const long long s = base + threadIdx.x;
  if (s >= n) return;
  const float4 a = sp[threadIdx.x + W];
  const float pa[3] = {a.x, a.y, a.z};
  float best = __int_as_float(0x7f800000);
#pragma unroll
  for (int k = 1; k <= W; ++k) {
#pragma unroll
    for (int sgn = -1; sgn <= 1; sgn += 2) {
      const float4 b = sp[threadIdx.x + W + sgn * k];
      if (b.x < __int_as_float(0x7f800000)) {
        const float pb[3] = {b.x, b.y, b.z};
        best = fminf(best, point_ub2<D>(pa, pb));
      }
    }
  }
  ub[s] = best < __int_as_float(0x7f800000)
              ? (unsigned long long)__double_as_longlong(__dmul_ru((double)__fsqrt_ru(best), 1.0 + 0x1p-40))
              : ~0ull;
}

// Round 1 of the solve: every slot is its own component (labels are the slot
// ids), so the boundary-pair fold of the round scan reduces to
// ub[s] = min(w(s-1, s), w(s, s+1)) (mst.py:198-224; f32 upper bounds of the weights, seed_weight):
// one streaming pass, no atomics, and no boundary prefix (round 1 labels no nodes).
template <int D>
__global__ void k_seed_round1(const float4* __restrict__ spts, long long n, const double* __restrict__ core,
                              unsigned long long* __restrict__ ub) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= n) return;
  const float4 a = spts[s];
  const float pa[3] = {a.x, a.y, a.z};
  double w = __longlong_as_double(0x7ff0000000000000ll);
  if (s > 0) {
    const float4 b = spts[s - 1];
    const float pb[3] = {b.x, b.y, b.z};
    double d = __longlong_as_double((long long)seed_weight<D>(pb, pa, false));   // (an upper bound suffices)
    if (core) d = fmax(d, fmax(core[s - 1], core[s]));
    w = d;
  }
  if (s + 1 < n) {
    const float4 b = spts[s + 1];
    const float pb[3] = {b.x, b.y, b.z};
    double d = __longlong_as_double((long long)seed_weight<D>(pa, pb, false));
    if (core) d = fmax(d, fmax(core[s], core[s + 1]));
    w = fmin(w, d);
  }
  ub[s] = s > 0 || s + 1 < n ? (unsigned long long)__double_as_longlong(w) : ~0ull;
}

// Extra radius seeds for the solve (not the reference's building block): slot
// s pairs with its Z-order neighbours s-W .. s+W (the direct neighbours are
// already in the boundary scan).  A pair in different components is a real
// outgoing edge, so its weight may lower both components' radii; only an upper
// bound is needed, so it is f32 rounded up (+2^-40 slack) -- no
// f64.  A block stages its slots [base, base+T) and W on either side (labels,
// points) in shared memory once.  Each pair (i, i+k), k = 1..W, is computed
// once, by the thread of its lower slot (including the W slots left of the
// block): the lower end keeps a register minimum, the upper end gets a
// shared-memory atomic min (squared f32 bounds >= 0 order as their bits).
// Every slot then sends one global atomic if it can lower its component's bound.
constexpr int kSeedThreads = 256;
constexpr int kSeedMaxW = 32;

template <int D, int kW>
__device__ __forceinline__ float seed_pairs(const float4* sp, const int* sl, unsigned* s_best, int a, int lim, int W) {
  const int la = sl[a];
  float mine = __int_as_float(0x7f800000);
  if (la < 0) return mine;
  const float4 pa = sp[a];
  const float q[3] = {pa.x, pa.y, pa.z};
  const int kmax = kW ? kW : W;
#pragma unroll
  for (int k = 1; k <= (kW ? kW : kSeedMaxW); ++k) {   // (k = 1: the boundary pairs; the scan then skips them)
    if (!kW && k > kmax) break;
    const int b = a + k;
    if (b >= lim) break;
    const int lb = sl[b];
    if (lb < 0 || lb == la) continue;
    const float4 pb = sp[b];
    const float p[3] = {pb.x, pb.y, pb.z};
    const float d2 = point_ub2<D>(q, p);
    mine = fminf(mine, d2);
    if (b >= W + 0 && b - W < kSeedThreads) atomicMin(&s_best[b - W], __float_as_uint(d2));
  }
  return mine;
}

template <int D, int kW>
__global__ void __launch_bounds__(kSeedThreads) k_seed_window(const int* __restrict__ label,
                                                              const float4* __restrict__ spts, long long n, int W,
                                                              unsigned long long* ub, long long block0 = 0) {
  // (block0: the first block of the launch -- a rank of a multi-GPU solve seeds the blocks
  // that cover its Morton range; every slot's seed comes from the block holding the slot)
  __shared__ float4 sp[kSeedThreads + 2 * kSeedMaxW];
  __shared__ int sl[kSeedThreads + 2 * kSeedMaxW];
  __shared__ unsigned s_best[kSeedThreads];
  if (kW) W = kW;
  const long long base = (block0 + blockIdx.x) * (long long)kSeedThreads;
  const int lim = kSeedThreads + 2 * W;
  for (int i = threadIdx.x; i < lim; i += kSeedThreads) {
    const long long g = base - W + i;
    const bool in = g >= 0 && g < n;
    sl[i] = in ? label[g] : -1;
    if (in) sp[i] = spts[g];
  }
  s_best[threadIdx.x] = 0x7f800000u;
  __syncthreads();
  // sources: staged slots [0, T + W) -- the left halo and the block itself
  const int me = threadIdx.x + W;
  float best2 = seed_pairs<D, kW>(sp, sl, s_best, me, lim, W);
  if (threadIdx.x < W) {
    const float h = seed_pairs<D, kW>(sp, sl, s_best, threadIdx.x, lim, W);   // halo source: upper ends only
    (void)h;
  }
  __syncthreads();
  best2 = fminf(best2, __uint_as_float(s_best[threadIdx.x]));
  const int ls = sl[me];
  unsigned long long w = best2 < __int_as_float(0x7f800000)
                             ? (unsigned long long)__double_as_longlong(__dmul_ru((double)__fsqrt_ru(best2), 1.0 + 0x1p-40))
                             : ~0ull;
  if (ls >= 0 && w != ~0ull && w < __ldcg(&ub[ls])) atomicMin(&ub[ls], w);
}

// ------------------------------------------------------------- node labels
// Reference semantics for every node (building blocks, subtree_skip off): a
// child's label is uniform iff no boundary falls in its slot range.
template <class Node>
__global__ void k_node_labels(Node* __restrict__ nodes, const int2* __restrict__ range, const int* __restrict__ bprefix,
                              const int* __restrict__ label, long long m) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= m) return;
  int2 r = range[i];
  const int2 refs = *reinterpret_cast<const int2*>(&nodes[i].ref.x);
  int gamma = refs.x >= 0 ? refs.x : ~refs.x;
  int bl = bprefix[r.x], bg = bprefix[gamma], bg1 = bprefix[gamma + 1], bh = bprefix[r.y];
  int ll = bg == bl ? label[r.x] : kMixed;
  int rl = bh == bg1 ? label[r.y] : kMixed;
  *reinterpret_cast<int2*>(&nodes[i].ref.z) = make_int2(ll, rl);
}

constexpr int kDirectFill = 128;   // top pure nodes up to this many slots fill top[] themselves

// top[s] = T + 1 for the top pure node T above slot s.  A top pure node (pure,
// mixed parent) is re-marked every round by its parent, and the top pure node of
// a slot only grows (pure stays pure), so filling the marked ranges each round
// keeps top[] exact without clearing it (0 = the slot's parent is mixed).
constexpr int kFillChunk = 1024;   // larger ones are cut into chunks of this many slots, a warp each

__device__ __forceinline__ void mark_top(int c, int lo, int hi, int* __restrict__ top, int4* __restrict__ big,
                                         unsigned* __restrict__ big_count) {
  if (hi - lo + 1 <= kDirectFill) {
    for (int s = lo; s <= hi; ++s) top[s] = c + 1;
  } else {
    const int k = (hi - lo + kFillChunk) / kFillChunk;
    const unsigned base = atomicAdd(big_count, (unsigned)k);
    for (int j = 0; j < k; ++j) {
      const int a = lo + j * kFillChunk;
      big[base + j] = make_int4(c + 1, a, min(hi, a + kFillChunk - 1), 0);
    }
  }
}

// the chunks of the larger ranges (disjoint: top pure nodes never nest), a warp per chunk
__global__ void k_fill_top(const int4* __restrict__ big, const unsigned* __restrict__ big_count,
                           int* __restrict__ top) {
  const unsigned cnt = *big_count;
  const unsigned lane = threadIdx.x & 31u;
  const unsigned warps = gridDim.x * (blockDim.x >> 5);
  for (unsigned w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < cnt; w += warps) {
    const int4 it = big[w];
    for (int s = it.y + (int)lane; s <= it.z; s += 32) top[s] = it.x;
  }
}

// Incremental labelling for the subtree-skip traversal.  A pure node stays
// pure (components only merge), and every query that reaches a node inside a
// pure subtree came from outside it, i.e. belongs to another component: for
// such visitors every child inside is foreign.  So when a node is found pure,
// its child labels become kInside (matches no component) once and for all, and
// only the nodes that were still mixed need looking at in later rounds.  A
// mixed node labels its children as before: MIXED, or the current id of a
// pure child (a top pure node, marked for the top[] scan as in k_node_labels).
// `list` = the nodes mixed last round (nullptr: all m nodes); the nodes still
// mixed are appended to out_list (warp-aggregated).
constexpr int kInside = -2;
constexpr int kLabelThreads = 256;   // k_node_labels_front block size (its append is per block)

template <class Node>
__global__ void k_node_labels_front(Node* __restrict__ nodes, const int2* __restrict__ range,
                                    const int* __restrict__ bprefix, const int* __restrict__ label,
                                    const int* __restrict__ list, long long count, int* __restrict__ out_list,
                                    unsigned* __restrict__ out_count, int* __restrict__ top, int4* __restrict__ big,
                                    unsigned* __restrict__ big_count) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool valid = t < count;
  const int i = valid ? (list ? list[t] : (int)t) : 0;
  bool mixed = false;
  if (valid) {
    const int2 r = range[i];
    const int4 ref4 = nodes[i].ref;   // child refs and the labels written last round
    const int2 refs = make_int2(ref4.x, ref4.y);
    const int gamma = refs.x >= 0 ? refs.x : ~refs.x;
    const int bl = bprefix[r.x], bh = bprefix[r.y];
    mixed = bl != bh;
    int2 lab = make_int2(kInside, kInside);
    if (mixed) {
      const int bg = bprefix[gamma], bg1 = bprefix[gamma + 1];
      lab.x = bg == bl ? label[r.x] : kMixed;
      lab.y = bh == bg1 ? label[r.y] : kMixed;
      // only a child that just turned pure is a new top pure node: one that was
      // already pure keeps its top[] entries from the round it turned pure
      if (top) {
        if (refs.x >= 0 && lab.x != kMixed && ref4.z == kMixed) mark_top(refs.x, r.x, gamma, top, big, big_count);
        if (refs.y >= 0 && lab.y != kMixed && ref4.w == kMixed) mark_top(refs.y, gamma + 1, r.y, top, big, big_count);
      }
    }
    // (a node that stays mixed with mixed children -- most of them early on --
    // keeps its labels: no write, so its record's sector is not dirtied)
    if (lab.x != ref4.z || lab.y != ref4.w) *reinterpret_cast<int2*>(&nodes[i].ref.z) = lab;
  }
  // one append per block: same-address atomics serialise at the L2 (~2-3 ns
  // each), and per-warp appends were ~840K of them in round 2 at 37M
  __shared__ unsigned s_off[kLabelThreads / 32];
  __shared__ unsigned s_base;
  const unsigned keep = __ballot_sync(0xffffffffu, mixed);
  const unsigned lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  if (lane == 0) s_off[wid] = __popc(keep);
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned run = 0;
    for (int w = 0; w < kLabelThreads / 32; ++w) { const unsigned c = s_off[w]; s_off[w] = run; run += c; }
    s_base = run ? atomicAdd(out_count, run) : 0u;
  }
  __syncthreads();
  if (mixed) out_list[s_base + s_off[wid] + __popc(keep & ((1u << lane) - 1u))] = i;
}

// Late rounds settle most queries before their first visit (nearest-foreign
// proof, top pure node, one-sided last round).  This pass applies the same
// tests as the traversal's query start, with the round's seeded radius (the
// radius only drops during the traversal, so every query dropped here would be
// dropped there too), and lists the slots left in Morton order -- per block of
// 256 slots, the blocks' runs in claim order -- so the traversal's warps run
// only real searches instead of cycling through settled queries.
template <int D>
__global__ void __launch_bounds__(kScanThreads) k_prefilter(const float4* __restrict__ spts, const int* __restrict__ label,
                                                            const unsigned long long* __restrict__ ub,
                                                            const float* __restrict__ nfn_lb, const int* __restrict__ top,
                                                            const int2* __restrict__ up, const Scene* __restrict__ scene_ptr,
                                                            long long q0, long long q1, const int* __restrict__ side,
                                                            int* __restrict__ out, unsigned* __restrict__ out_count,
                                                            unsigned long long* __restrict__ skipped) {
  // a thread owns kScanItems consecutive slots of a kScanTile-slot tile; one
  // list append (atomic) per tile, the tile's kept slots in Morton order
  __shared__ unsigned s_base;
  const Scene sc = *scene_ptr;
  const int skip_comp = side ? *side : -1;
  unsigned long long nskip = 0;
  for (long long t0 = q0 + (long long)blockIdx.x * kScanTile; t0 < q1; t0 += (long long)gridDim.x * kScanTile) {
    const long long i0 = t0 + (long long)threadIdx.x * kScanItems;
    unsigned keep = 0;   // bit j: slot i0 + j is listed
    // the thread's 8 labels, proofs and top pure nodes in 16-byte loads (a
    // shard range may start off the 8-slot grid: those tiles load per slot)
    const int cnt = i0 >= q1 ? 0 : (q1 - i0 < kScanItems ? (int)(q1 - i0) : kScanItems);
    const int vcnt = (i0 & (kScanItems - 1)) ? -1 : cnt;
    int labs[kScanItems], tops[kScanItems];
    float lbs[kScanItems];
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) { labs[j] = 0; tops[j] = 0; lbs[j] = 0.f; }
    if (vcnt >= 0) {
      load8(label, i0, vcnt, labs);
      load8(nfn_lb, i0, vcnt, lbs);
      if (top) load8(top, i0, vcnt, tops);
    } else {
#pragma unroll
      for (int j = 0; j < kScanItems; ++j)
        if (j < cnt) { labs[j] = label[i0 + j]; lbs[j] = nfn_lb[i0 + j]; tops[j] = top ? top[i0 + j] : 0; }
    }
    // (the bounds are final here: read through L1, once per run of equal labels)
    int plab = -1;
    double prad = 0.0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
      const long long s = i0 + j;
      if (j >= cnt) break;
      const int comp = labs[j];
      const double radius = comp == plab ? prad : bits_to_radius(__ldg(&ub[comp]));
      plab = comp;
      prad = radius;
      bool k = !((double)lbs[j] > radius) && comp != skip_comp;
      if (k && top) {
        const int t = tops[j];
        if (t > 0) {
          const int2 ut = __ldg(up + (t - 1));
          if (ut.x < 0) {
            k = false;
          } else if (radius < 1e300) {
            const float4 pv = spts[s];
            const float q[3] = {pv.x, pv.y, pv.z};
            if (ut.y <= ball_prefix<D>(q, radius, sc)) k = false;
          }
        }
      }
      keep |= (unsigned)k << j;
      nskip += !k;
    }
    unsigned total;
    const unsigned off = block_exclusive<unsigned>(__popc(keep), &total);
    if (threadIdx.x == 0) s_base = total ? atomicAdd(out_count, total) : 0u;
    __syncthreads();
    unsigned pos = s_base + off;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j)
      if (keep >> j & 1u) out[pos++] = (int)(i0 + j);
    __syncthreads();   // (s_base is rewritten by the next tile)
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nskip += __shfl_xor_sync(0xffffffffu, nskip, o);
  if ((threadIdx.x & 31u) == 0 && nskip) atomicAdd(skipped, nskip);
}

// slots whose label is `value` (warp-aggregated)
__global__ void k_count_label(const int* __restrict__ label, long long n, int value, unsigned long long* __restrict__ out) {
  unsigned long long cnt = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    cnt += label[i] == value;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31u) == 0 && cnt) atomicAdd(out, cnt);
}

// the larger of the last two components (slots of component 1 vs n): its queries are not run
__global__ void k_pick_side(const unsigned long long* __restrict__ count1, long long n, int* __restrict__ side) {
  if (threadIdx.x == 0) *side = 2 * (long long)*count1 > n ? 1 : 0;
}

// the two components of the last round share their minimum edge: copy it to the side left out
__global__ void k_copy_key(EdgeKey* best, const int* __restrict__ side) {
  if (threadIdx.x == 0) {
    const int s = *side;
    best[s] = best[1 - s];
  }
}

// ------------------------------------------------------------------- merge
constexpr int kErrNoEdge = 1;     // mst.py:365-376 / 720-721
constexpr int kErrChain = 2;      // mst.py:399-400 / 722-723

__global__ void k_merge_succ(const EdgeKey* __restrict__ best, long long c, const int* __restrict__ label,
                             const unsigned* __restrict__ perm, const unsigned* __restrict__ iperm,
                             int* __restrict__ succ, int* __restrict__ err, bool singletons) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= c) return;
  EdgeKey e = best[k];
  if (e.uv == ~0ull) { atomicOr(err, kErrNoEdge); succ[k] = (int)k; return; }
  unsigned u = (unsigned)(e.uv >> 32), v = (unsigned)(e.uv & 0xffffffffu);
  int su, sv;
  if (singletons) {
    // round 1: every slot is its own component (label[s] == s) and one end of
    // its edge is its own point perm[k]: only the other end is looked up
    const unsigned pk = perm[k];
    su = u == pk ? (int)k : (int)iperm[u];
    sv = v == pk ? (int)k : (int)iperm[v];
  } else {
    su = (int)iperm[u];
    sv = (int)iperm[v];
  }
  int lu = singletons ? su : label[su], lv = singletons ? sv : label[sv];
  if (lu == (int)k && lv != (int)k) succ[k] = lv;
  else if (lv == (int)k && lu != (int)k) succ[k] = lu;
  else { atomicOr(err, kErrNoEdge); succ[k] = (int)k; }
}

// Each component points at its successor; the smaller member of a mutual pair
// points at itself and becomes the cluster root (mst.py:385-402).
__global__ void k_merge_link(const int* __restrict__ succ, long long c, int* __restrict__ ptr) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= c) return;
  int y = succ[k];
  ptr[k] = succ[y] == (int)k ? min((int)k, y) : y;
}

// Find-with-path-halving to the root; concurrent halving only ever replaces a
// pointer with one of its ancestors, so racing threads stay correct.  The
// result goes to root[k], which only thread k writes (ptr[k] itself may still
// be overwritten by another thread's halving step).
__global__ void k_merge_jump(int* ptr, long long c, int* __restrict__ root, int* __restrict__ err) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= c) return;
  volatile int* vp = ptr;
  int x = (int)k;
  long long steps = 0;
  for (;;) {
    int p = vp[x];
    if (p == x) break;
    int pp = vp[p];
    if (pp != p) vp[x] = pp;
    x = pp;
    if (++steps > c) { atomicOr(err, kErrChain); break; }
  }
  root[k] = x;
}

// flags packed for one scan: bits 0..30 "emits its edge" (mst.py:416-423),
// bits 31..61 "is a cluster root"; the store appends the emitted edges and
// gives every root its new dense id.
struct MergeScanOp {
  using T = unsigned long long;
  static constexpr bool kCached = true;   // the scan pass reads the flags the reduce pass cached
  __device__ void side(long long, int, const unsigned long long*) const {}
  const int* succ;
  const int* root;
  const EdgeKey* best;
  EdgeKey* eout;   // emitted edges (u << 32 | v, weight bits), one 16-byte record each
  long long edge_base;
  int* newid;
  unsigned char* cache;   // one byte of flags per component (bit 0 edge, bit 1 root), 8-aligned runs
  // The flags need a random read (succ[succ[k]]); the reduce pass caches them so
  // that the scan pass reads 1 coalesced byte per component instead.
  __device__ void put(long long i0, int cnt, const unsigned long long* v) const {
    unsigned long long b = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j)
      if (j < cnt) b |= (unsigned long long)((v[j] & 1ull) | ((v[j] >> 30) & 2ull)) << (8 * j);
    if (cnt == kScanItems) *reinterpret_cast<unsigned long long*>(cache + i0) = b;
    else
      for (int j = 0; j < cnt; ++j) cache[i0 + j] = (unsigned char)(b >> (8 * j));
  }
  __device__ void get(long long i0, int cnt, unsigned long long* v) const {
    unsigned long long b = 0;
    if (cnt == kScanItems) b = *reinterpret_cast<const unsigned long long*>(cache + i0);
    else
      for (int j = 0; j < cnt; ++j) b |= (unsigned long long)cache[i0 + j] << (8 * j);
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
      const unsigned long long f = (b >> (8 * j)) & 3ull;
      v[j] = j < cnt ? ((f & 1ull) | ((f >> 1) << 31)) : 0ull;
    }
  }
  __device__ void load(long long i0, int cnt, unsigned long long* v) const {
    int y[kScanItems], r[kScanItems], yy[kScanItems];
    load8(succ, i0, cnt, y);
    load8(root, i0, cnt, r);
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) yy[j] = j < cnt ? __ldg(succ + y[j]) : -1;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
      if (j >= cnt) continue;
      const int k = (int)(i0 + j);
      const bool mutual = yy[j] == k;
      const unsigned long long edge = (mutual && y[j] < k) ? 0ull : 1ull;
      const unsigned long long is_root = r[j] == k ? 1ull : 0ull;
      v[j] = edge | (is_root << 31);
    }
  }
  // Called by every thread (cnt may be 0).  The edge records move warp-striped:
  // each thread parks its 8 output positions in shared memory, then lane l
  // copies items l, l + 32, ... of the warp's 256, so a warp's 16-byte reads of
  // best and writes to eout are contiguous instead of 128 bytes apart.
  static constexpr bool kWarpStore = true;
  __device__ void store(long long i0, int cnt, const unsigned long long* v, unsigned long long ex) const {
    __shared__ int4 s_pos4[kScanThreads * kScanItems / 4];
    int pos[kScanItems];
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
      pos[j] = -1;
      if (j >= cnt) continue;
      if (v[j] & 1ull) pos[j] = (int)(ex & 0x7fffffffull);
      if (v[j] >> 31) newid[i0 + j] = (int)(ex >> 31);
      ex += v[j];
    }
    const unsigned lane = threadIdx.x & 31u;
    int4* mine = s_pos4 + threadIdx.x * (kScanItems / 4);
    mine[0] = make_int4(pos[0], pos[1], pos[2], pos[3]);
    mine[1] = make_int4(pos[4], pos[5], pos[6], pos[7]);
    __syncwarp();
    const int* wpos = reinterpret_cast<const int*>(s_pos4) + (threadIdx.x - lane) * kScanItems;
    const long long w0 = i0 - (long long)lane * kScanItems;   // the warp's first item
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
      const int idx = j * 32 + (int)lane;
      const int at = wpos[idx];
      if (at >= 0) eout[edge_base + at] = best[w0 + idx];
    }
    __syncwarp();   // (the positions are rewritten by the next tile)
  }
};

__global__ void k_merge_final(const int* __restrict__ root, const int* __restrict__ newid, long long c, int* __restrict__ fin) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= c) return;
  fin[k] = newid[root[k]];
}

// 4 slots per thread with 16-byte accesses (label is a cudaMalloc'd array: aligned)
__global__ void k_relabel(int* __restrict__ label, const int* __restrict__ fin, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long s = i << 2;
  if (s + 3 < n) {
    int4 v = reinterpret_cast<const int4*>(label)[i];
    v.x = __ldg(fin + v.x); v.y = __ldg(fin + v.y); v.z = __ldg(fin + v.z); v.w = __ldg(fin + v.w);
    reinterpret_cast<int4*>(label)[i] = v;
  } else {
    for (long long t = s; t < n; ++t) label[t] = fin[label[t]];
  }
}

// ---------------------------------------------------- multi-shard exchange
// Two-phase (w, then uv) min so that a u64 min-allreduce is exact for the
// 128-bit (w, u, v) order.
__global__ void k_split_keys(const EdgeKey* __restrict__ best, long long c, unsigned long long* __restrict__ w) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k < c) w[k] = best[k].w;
}
__global__ void k_mask_uv(const EdgeKey* __restrict__ best, const unsigned long long* __restrict__ wmin, long long c,
                          unsigned long long* __restrict__ uv) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= c) return;
  EdgeKey e = best[k];
  uv[k] = e.w == wmin[k] ? e.uv : ~0ull;
}
__global__ void k_join_keys(EdgeKey* __restrict__ best, const unsigned long long* __restrict__ wmin,
                            const unsigned long long* __restrict__ uvmin, long long c) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= c) return;
  EdgeKey e;
  e.w = wmin[k];
  e.uv = uvmin[k];
  best[k] = e;
}
// Folds rows 1..rows-1 of `buf` (row stride `stride`) into row 0 by min or sum:
// the local (virtual-shard) stage of the exchange's all-reduce.
__global__ void k_fold_rows(unsigned long long* __restrict__ buf, int rows, long long stride, long long c, bool sum) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= c) return;
  unsigned long long a = buf[k];
  for (int g = 1; g < rows; ++g) {
    const unsigned long long b = buf[g * stride + k];
    a = sum ? a + b : min(a, b);
  }
  buf[k] = a;
}

// ------------------------------------------------------------ final output
// The (w, u, v) order of the n - 1 edges (mst.py:745-747) in two steps:
//   1. a stable 4-pass radix sort on a 32-bit key: the weight bits minus the
//      smallest weight's bits, shifted right just enough to fit 32 bits
//      (monotone in w >= 0: w_a < w_b implies key_a <= key_b; at 37M blobs 3D
//      one key spans 2^24 f64 ulps, a relative 2^-28);
//   2. every run of equal keys (true ties and the rare collisions) is put in
//      exact (w bits, u << 32 | v) order -- 128-bit keys, all distinct.
// Edges live as one 16-byte record (uv, w) so that every gather is one sector.
constexpr int kThreadTie = 8;     // tie runs up to this long are ordered in registers by one thread
constexpr int kShortTie = 32;     // ... up to this long by one warp each
constexpr int kSmallTie = 256;    // ... up to this long by one 128-thread block each (small shared footprint)
constexpr int kBlockTie = 4096;   // longer ones up to this long by one block each

// range[0] = min, range[1] = max of the weight bits (range preset to (~0, 0))
__global__ void __launch_bounds__(256) k_edge_wrange(const EdgeKey* __restrict__ e, long long ne,
                                                     unsigned long long* __restrict__ range) {
  unsigned long long lo = ~0ull, hi = 0ull;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < ne; i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long w = e[i].w;
    lo = min(lo, w);
    hi = max(hi, w);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(range, lo);
    atomicMax(range + 1, hi);
  }
}

__device__ __forceinline__ int wkey_shift(const unsigned long long* range) {
  const unsigned long long span = range[1] - range[0];
  const int bits = span ? 64 - __clzll((long long)span) : 0;
  return bits > 32 ? bits - 32 : 0;
}

// the 32-bit sort key of each emitted edge
__global__ void k_edge_wkey(const EdgeKey* __restrict__ e, long long ne, const unsigned long long* __restrict__ range,
                            unsigned* __restrict__ key) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < ne) key[i] = (unsigned)((e[i].w - range[0]) >> wkey_shift(range));
}

__device__ __forceinline__ bool wuv_less(const EdgeKey& a, const EdgeKey& b) {
  return a.w < b.w || (a.w == b.w && a.uv < b.uv);
}

// One pass over the key-sorted edges.  The thread at the start of each run of
// equal keys measures it and puts it into exact (w, u, v) order: a run of at
// most kThreadTie edges itself, in registers; a longer one of at most kShortTie
// is listed in `mid` for a warp (k_edge_fix_mid), one of at most kBlockTie in
// `runs` for a block (k_edge_fix_long), as (start, length); a still longer run
// raises *max_run above kBlockTie and the host redoes the order with the exact
// two-key sort.
__global__ void k_edge_ties(const unsigned* __restrict__ key, long long ne, const EdgeKey* __restrict__ eout,
                            unsigned* __restrict__ order, unsigned* __restrict__ max_run, int2* __restrict__ runs,
                            unsigned* __restrict__ run_count, int2* __restrict__ mid, unsigned* __restrict__ mid_count,
                            int2* __restrict__ small, unsigned* __restrict__ small_count) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int len = 0;
  if (i + 1 < ne) {
    const unsigned ki = key[i];
    if (ki == key[i + 1] && (i == 0 || key[i - 1] != ki)) {   // a run starts here
      // run length by galloping + binary search (the keys are sorted), capped at kBlockTie + 1
      const long long cap = min(ne, i + kBlockTie + 1);   // positions [i, cap) may belong to the run
      long long lo = i + 1, hi = i + 2;                   // key[lo] == ki; hi: first candidate to test
      while (hi < cap && key[hi] == ki) {
        lo = hi;
        hi = min(cap, i + 2 * (hi - i));
      }
      while (hi - lo > 1) {   // last equal position in [lo, hi)
        const long long m = (lo + hi) >> 1;
        if (key[m] == ki) lo = m; else hi = m;
      }
      len = (int)(lo - i + 1);
    }
  }
  // (a run of exactly two is ordered by the emit itself, which gathers both records anyway)
  if (len > 2 && len <= kThreadTie) {
    // in registers: all loads issued at once, then a fixed compare-exchange network
    unsigned o[kThreadTie];
    EdgeKey k[kThreadTie];
#pragma unroll
    for (int a = 0; a < kThreadTie; ++a) o[a] = a < len ? order[i + a] : 0u;
#pragma unroll
    for (int a = 0; a < kThreadTie; ++a) {
      if (a < len) k[a] = eout[o[a]];
      else { k[a].w = ~0ull; k[a].uv = ~0ull; }
    }
#pragma unroll
    for (int a = 1; a < kThreadTie; ++a) {
#pragma unroll
      for (int b = a; b > 0; --b) {
        if (wuv_less(k[b], k[b - 1])) {
          const EdgeKey t = k[b - 1]; k[b - 1] = k[b]; k[b] = t;
          const unsigned u = o[b - 1]; o[b - 1] = o[b]; o[b] = u;
        }
      }
    }
#pragma unroll
    for (int a = 0; a < kThreadTie; ++a) if (a < len) order[i + a] = o[a];
  } else if (len > kBlockTie) {
    atomicMax(max_run, (unsigned)len);   // (only the overflow matters to the host)
  } else if (len > kSmallTie) {
    runs[atomicAdd(run_count, 1u)] = make_int2((int)i, len);
  } else if (len > kShortTie) {
    small[atomicAdd(small_count, 1u)] = make_int2((int)i, len);
  }
  // runs of kThreadTie+1..kShortTie: one list append per warp
  const bool is_mid = len > kThreadTie && len <= kShortTie;
  const unsigned m = __ballot_sync(0xffffffffu, is_mid);
  if (m) {
    const unsigned lane = threadIdx.x & 31u;
    const int leader = __ffs(m) - 1;
    unsigned base = 0;
    if ((int)lane == leader) base = atomicAdd(mid_count, (unsigned)__popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (is_mid) mid[base + __popc(m & ((1u << lane) - 1u))] = make_int2((int)i, len);
  }
}

// A warp per listed run of kThreadTie+1..kShortTie edges: bitonic sort of
// ((w, uv), edge) across the lanes.  Grid-stride over the device-side count.
__global__ void k_edge_fix_mid(const int2* __restrict__ mid, const unsigned* __restrict__ mid_count,
                               const EdgeKey* __restrict__ eout, unsigned* __restrict__ order) {
  const unsigned cnt = *mid_count;
  const int lane = (int)(threadIdx.x & 31u);
  const unsigned warps = gridDim.x * (blockDim.x >> 5);
  for (unsigned r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < cnt; r += warps) {
    const int2 run = mid[r];
    unsigned o = 0;
    EdgeKey k;
    k.w = ~0ull;
    k.uv = ~0ull;
    if (lane < run.y) {
      o = order[run.x + lane];
      k = eout[o];
    }
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
      for (int j = size >> 1; j > 0; j >>= 1) {
        EdgeKey p;
        p.w = __shfl_xor_sync(0xffffffffu, k.w, j);
        p.uv = __shfl_xor_sync(0xffffffffu, k.uv, j);
        const unsigned po = __shfl_xor_sync(0xffffffffu, o, j);
        const bool lower = (lane & j) == 0;
        const bool up = (lane & size) == 0;
        // the lower lane of a pair keeps the min when sorting up, the max otherwise
        const bool take = lower == up ? wuv_less(p, k) : wuv_less(k, p);
        if (take) { k = p; o = po; }
      }
    }
    if (lane < run.y) order[run.x + lane] = o;
  }
}

// One 128-thread block per listed run of kShortTie+1..kSmallTie edges (grid-stride over the
// device-side count): the same bitonic sort as k_edge_fix_long in 5 KB of shared memory, so many
// blocks share an SM and a short run does not hold a 1024-thread block through its barriers.
constexpr int kSmallTieThreads = 128;
__global__ void __launch_bounds__(kSmallTieThreads) k_edge_fix_small(const int2* __restrict__ runs,
                                                                     const unsigned* __restrict__ run_count,
                                                                     const EdgeKey* __restrict__ eout,
                                                                     unsigned* __restrict__ order) {
  __shared__ EdgeKey sk[kSmallTie];
  __shared__ unsigned so[kSmallTie];
  const unsigned cnt = *run_count;
  for (unsigned ri = blockIdx.x; ri < cnt; ri += gridDim.x) {
    const int2 r = runs[ri];
    int size = 1;
    while (size < r.y) size <<= 1;
    for (int a = threadIdx.x; a < size; a += blockDim.x) {
      const unsigned o = a < r.y ? order[r.x + a] : 0u;
      so[a] = o;
      if (a < r.y) sk[a] = eout[o];
      else { sk[a].w = ~0ull; sk[a].uv = ~0ull; }
    }
    __syncthreads();
    for (int k = 2; k <= size; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int a = threadIdx.x; a < size; a += blockDim.x) {
          const int b = a ^ j;
          if (b > a) {
            const bool up = (a & k) == 0;
            const EdgeKey ka = sk[a], kb = sk[b];
            if (wuv_less(kb, ka) == up) {
              sk[a] = kb; sk[b] = ka;
              const unsigned t = so[a]; so[a] = so[b]; so[b] = t;
            }
          }
        }
        __syncthreads();
      }
    }
    for (int a = threadIdx.x; a < r.y; a += blockDim.x) order[r.x + a] = so[a];
    __syncthreads();   // (the shared arrays are reused by the next run)
  }
}

// One block per listed run (kSmallTie < length <= kBlockTie; grid-stride over
// the device-side count): bitonic sort of the run's ((w, uv), edge) triples in
// shared memory (dynamic, kEdgeFixSmem bytes).
constexpr size_t kEdgeFixSmem = (size_t)kBlockTie * (16 + 4);
__global__ void __launch_bounds__(1024) k_edge_fix_long(const int2* __restrict__ runs,
                                                        const unsigned* __restrict__ run_count,
                                                        const EdgeKey* __restrict__ eout,
                                                        unsigned* __restrict__ order) {
  extern __shared__ __align__(16) unsigned char fix_smem[];
  EdgeKey* sk = reinterpret_cast<EdgeKey*>(fix_smem);
  unsigned* so = reinterpret_cast<unsigned*>(sk + kBlockTie);
  const unsigned cnt = *run_count;
  for (unsigned ri = blockIdx.x; ri < cnt; ri += gridDim.x) {
    const int2 r = runs[ri];
    int size = 1;
    while (size < r.y) size <<= 1;
    for (int a = threadIdx.x; a < size; a += blockDim.x) {
      const unsigned o = a < r.y ? order[r.x + a] : 0u;
      so[a] = o;
      if (a < r.y) sk[a] = eout[o];
      else { sk[a].w = ~0ull; sk[a].uv = ~0ull; }
    }
    __syncthreads();
    for (int k = 2; k <= size; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int a = threadIdx.x; a < size; a += blockDim.x) {
          const int b = a ^ j;
          if (b > a) {
            const bool up = (a & k) == 0;
            const EdgeKey ka = sk[a], kb = sk[b];
            if (wuv_less(kb, ka) == up) {
              sk[a] = kb; sk[b] = ka;
              const unsigned t = so[a]; so[a] = so[b]; so[b] = t;
            }
          }
        }
        __syncthreads();
      }
    }
    for (int a = threadIdx.x; a < r.y; a += blockDim.x) order[r.x + a] = so[a];
    __syncthreads();   // (the shared arrays are reused by the next run)
  }
}

// the exact fallback's keys: uv of each edge, then its weight bits in a given order
__global__ void k_edge_uv_keys(const EdgeKey* __restrict__ eout, long long ne, unsigned long long* __restrict__ keys) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < ne) keys[i] = eout[i].uv;
}
__global__ void k_edge_w_keys(const EdgeKey* __restrict__ eout, const unsigned* __restrict__ order, long long ne,
                              unsigned long long* __restrict__ keys) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < ne) keys[i] = eout[order[i]].w;
}

// The record at final position i.  With the sorted 32-bit keys given, a run of
// exactly two equal keys (the common tie or collision, left alone by
// k_edge_ties) is put in exact (w, uv) order here: its first position takes the
// smaller of the two records, its second the larger (the partner's record by
// shuffle, or loaded at a warp edge).  All lanes of the warp must call it.
// (i1: the end of the launch's positions, <= ne; a partner outside [i0, i1) is loaded)
__device__ __forceinline__ EdgeKey final_record(const unsigned* __restrict__ order, const EdgeKey* __restrict__ eout,
                                                const unsigned* __restrict__ key, long long ne, long long i,
                                                long long i0, long long i1) {
  const bool valid = i < i1;
  EdgeKey e;
  e.w = ~0ull;
  e.uv = ~0ull;
  if (valid) e = eout[order[i]];
  if (!key) return e;   // (grid-uniform: the exact fallback's order has no ties left)
  int side = 0;         // +1: first of a two-run, -1: its second
  if (valid) {
    const unsigned k0 = key[i];
    const bool eqn = i + 1 < ne && key[i + 1] == k0, eqp = i > 0 && key[i - 1] == k0;
    if (eqn && !eqp && !(i + 2 < ne && key[i + 2] == k0)) side = 1;
    else if (eqp && !eqn && !(i > 1 && key[i - 2] == k0)) side = -1;
  }
  const unsigned lane = threadIdx.x & 31u;
  EdgeKey up, dn;   // the records of lanes + 1 and - 1
  up.w = __shfl_down_sync(0xffffffffu, e.w, 1);
  up.uv = __shfl_down_sync(0xffffffffu, e.uv, 1);
  dn.w = __shfl_up_sync(0xffffffffu, e.w, 1);
  dn.uv = __shfl_up_sync(0xffffffffu, e.uv, 1);
  if (side == 1) {
    const EdgeKey p = lane == 31 || i + 1 >= i1 ? eout[order[i + 1]] : up;
    if (wuv_less(p, e)) e = p;
  } else if (side == -1) {
    const EdgeKey p = lane == 0 || i - 1 < i0 ? eout[order[i - 1]] : dn;
    if (wuv_less(e, p)) e = p;
  }
  return e;
}

// edge order -> the reference's int64 (u, v) rows and f64 weights
__global__ void k_edge_emit(const unsigned* __restrict__ order, const EdgeKey* __restrict__ eout,
                            const unsigned* __restrict__ key, long long ne, long long* __restrict__ edges,
                            double* __restrict__ weights) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const EdgeKey e = final_record(order, eout, key, ne, i, 0, ne);
  if (i >= ne) return;
  reinterpret_cast<longlong2*>(edges)[i] = make_longlong2((long long)(e.uv >> 32), (long long)(e.uv & 0xffffffffull));
  weights[i] = __longlong_as_double((long long)e.w);
}

// the host-pointer entry's variant: packed (u << 32 | v) rows, 8 bytes per edge over PCIe (hostio.h)
// (positions [i0, i1): the host-output path emits in chunks, each one's copy starting behind it)
__global__ void k_edge_emit_packed(const unsigned* __restrict__ order, const EdgeKey* __restrict__ eout,
                                   const unsigned* __restrict__ key, long long ne,
                                   unsigned long long* __restrict__ packed, double* __restrict__ weights,
                                   long long i0, long long i1) {
  const long long i = i0 + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const EdgeKey e = final_record(order, eout, key, ne, i, i0, i1);
  if (i >= i1) return;
  packed[i] = e.uv;
  weights[i] = __longlong_as_double((long long)e.w);
}

// ----------------------------------------------------- total weight (numpy order)
// float(np.sum(weights)) (mst.py:749) reproduced bit for bit: numpy adds a
// float64 array by pairwise summation -- blocks of <= 128 with 8 interleaved
// accumulators combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a
// sequential tail, longer ranges split at n/2 rounded down to a multiple of 8
// -- and the reduction starts from 0.0 (numpy loops_utils.h.src pairwise_sum).
// The recursion tree depends on n only, so the 2^L subtrees at depth L are
// summed by one thread each and their results combined level by level in the
// same order.  All adds are _rn (no contraction).
constexpr int kPairwiseLevels = 16;   // up to 65536 partial sums (every node above depth L splits when n >= 256 * 2^L)
constexpr int kCombineLevels = 12;    // levels one block combines (4096 values in shared memory)

__device__ double pairwise_block(const double* a, long long n) {
  if (n < 8) {
    double res = 0.0;
    for (long long i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  long long i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, a[i]);
  return res;
}

__device__ double pairwise_sum(const double* a, long long n) {
  if (n <= 128) return pairwise_block(a, n);
  long long n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pairwise_sum(a, n2), pairwise_sum(a + n2, n - n2));
}

// Subtree `t` at depth `levels` of the split recursion over [0, n): follow the
// bits of t from the most significant (0 = first half).
__global__ void k_pairwise_partials(const double* __restrict__ a, long long n, int levels, double* __restrict__ part) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (1 << levels)) return;
  long long off = 0, len = n;
  for (int l = levels - 1; l >= 0; --l) {
    long long n2 = len / 2;
    n2 -= n2 % 8;
    if ((t >> l) & 1) { off += n2; len -= n2; } else { len = n2; }
  }
  part[t] = pairwise_sum(a + off, len);
}

// Block b combines the 2^g values part[b * 2^g ..] pairwise, level by level
// (a depth-g subtree of the recursion), into out[b]; `zero` adds the final 0.0.
__global__ void k_pairwise_combine(const double* __restrict__ part, int g, double* __restrict__ out, bool zero) {
  __shared__ double s[1 << kCombineLevels];
  const double* p = part + ((long long)blockIdx.x << g);
  for (int i = threadIdx.x; i < (1 << g); i += blockDim.x) s[i] = p[i];
  __syncthreads();
  for (int l = g; l > 0; --l) {
    const int half = 1 << (l - 1);
    double v[(1 << kCombineLevels) / 2 / 1024];
#pragma unroll
    for (int k = 0; k < (1 << kCombineLevels) / 2 / 1024; ++k) {
      const int i = threadIdx.x + k * 1024;
      v[k] = i < half ? __dadd_rn(s[2 * i], s[2 * i + 1]) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < (1 << kCombineLevels) / 2 / 1024; ++k) {
      const int i = threadIdx.x + k * 1024;
      if (i < half) s[i] = v[k];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = zero ? __dadd_rn(0.0, s[0]) : s[0];
}

}  // namespace emst
