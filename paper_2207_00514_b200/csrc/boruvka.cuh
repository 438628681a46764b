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
struct RoundScanLoad {
  const int* label;
  const float4* spts;
  unsigned long long* ub;
  long long n;
  int dim;
  bool bounds;
  __device__ unsigned long long operator()(long long i) const {
    if (i + 1 >= n) return 0ull;
    int la = label[i], lb = label[i + 1];
    if (la == lb) return 0ull;
    if (bounds) {
      float4 a = spts[i], b = spts[i + 1];
      float pa[3] = {a.x, a.y, a.z}, pb[3] = {b.x, b.y, b.z};
      double w = dim == 3 ? exact_dist<3>(pa, pb) : exact_dist<2>(pa, pb);
      unsigned long long bits = (unsigned long long)__double_as_longlong(w);
      // late rounds funnel many boundary pairs into few components: read first,
      // and only issue the atomic when it can still lower the bound
      if (bits < __ldcg(&ub[la])) atomicMin(&ub[la], bits);
      if (bits < __ldcg(&ub[lb])) atomicMin(&ub[lb], bits);
    }
    return 1ull;
  }
};
struct RoundScanStore {
  int* bprefix;
  __device__ void operator()(long long i, unsigned long long excl) const { bprefix[i] = (int)excl; }
};

// ------------------------------------------------------------- node labels
// Also marks the "top pure" nodes: an internal child whose slot range lies in
// one component while the node itself is mixed.  Every leaf under such a node T
// has T as its highest single-component ancestor; the marks (T + 1 at the first
// and the last slot of T's range) are turned into top[s] by k_scan<TopScan*>.
template <class Node>
__global__ void k_node_labels(Node* __restrict__ nodes, const int2* __restrict__ range, const int* __restrict__ bprefix,
                              const int* __restrict__ label, long long m, int* __restrict__ mark_lo,
                              int* __restrict__ mark_hi) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= m) return;
  int2 r = range[i];
  const int2 refs = *reinterpret_cast<const int2*>(&nodes[i].ref.x);
  int gamma = refs.x >= 0 ? refs.x : ~refs.x;
  int bl = bprefix[r.x], bg = bprefix[gamma], bg1 = bprefix[gamma + 1], bh = bprefix[r.y];
  int ll = bg == bl ? label[r.x] : kMixed;
  int rl = bh == bg1 ? label[r.y] : kMixed;
  *reinterpret_cast<int2*>(&nodes[i].ref.z) = make_int2(ll, rl);
  if (mark_lo && bl != bh) {
    if (refs.x >= 0 && ll != kMixed) { mark_lo[r.x] = refs.x + 1; mark_hi[gamma] = refs.x + 1; }
    if (refs.y >= 0 && rl != kMixed) { mark_lo[gamma + 1] = refs.y + 1; mark_hi[r.y] = refs.y + 1; }
  }
}

// top[s] = T + 1 for the top pure node T whose range holds slot s, else 0.  The
// ranges are disjoint, so top[s] = sum_{j <= s} mark_lo[j] - sum_{j < s} mark_hi[j]:
// an exclusive scan of (mark_lo - mark_hi) plus mark_lo[s], in u64 arithmetic
// that is exact modulo 2^62 (the scan keeps 62 value bits).  The store clears
// the marks for the next round (each index is read and cleared by one thread).
struct TopScanLoad {
  const int* mark_lo;
  const int* mark_hi;
  __device__ unsigned long long operator()(long long i) const {
    return (unsigned long long)(unsigned)mark_lo[i] - (unsigned long long)(unsigned)mark_hi[i];
  }
};
struct TopScanStore {
  int* mark_lo;
  int* mark_hi;
  int* top;
  __device__ void operator()(long long i, unsigned long long excl) const {
    const int lo = mark_lo[i], hi = mark_hi[i];
    top[i] = (int)((excl + (unsigned long long)(unsigned)lo) & kValueMask);
    if (lo) mark_lo[i] = 0;
    if (hi) mark_hi[i] = 0;
  }
};

// ------------------------------------------------------------------- merge
constexpr int kErrNoEdge = 1;     // mst.py:365-376 / 720-721
constexpr int kErrChain = 2;      // mst.py:399-400 / 722-723

__global__ void k_merge_succ(const EdgeKey* __restrict__ best, long long c, const int* __restrict__ label,
                             const unsigned* __restrict__ iperm, int* __restrict__ succ, int* __restrict__ err) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= c) return;
  EdgeKey e = best[k];
  if (e.uv == ~0ull) { atomicOr(err, kErrNoEdge); succ[k] = (int)k; return; }
  unsigned u = (unsigned)(e.uv >> 32), v = (unsigned)(e.uv & 0xffffffffu);
  int lu = label[iperm[u]], lv = label[iperm[v]];
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

// flags packed for one scan: bit 0..30 "emits its edge", bit 31.. "is a root"
struct MergeScanLoad {
  const int* succ;
  const int* root;
  __device__ unsigned long long operator()(long long k) const {
    int y = succ[k];
    bool mutual = succ[y] == (int)k;
    unsigned long long edge = (mutual && y < (int)k) ? 0ull : 1ull;   // mst.py:416-423
    unsigned long long is_root = root[k] == (int)k ? 1ull : 0ull;
    return edge | (is_root << 31);
  }
};
struct MergeScanStore {
  const int* succ;
  const int* root;
  const EdgeKey* best;
  unsigned* eu;
  unsigned* ev;
  unsigned long long* ew;
  long long edge_base;
  int* newid;
  __device__ void operator()(long long k, unsigned long long excl) const {
    int y = succ[k];
    bool mutual = succ[y] == (int)k;
    if (!(mutual && y < (int)k)) {
      long long at = edge_base + (long long)(excl & 0x7fffffffull);
      EdgeKey e = best[k];
      eu[at] = (unsigned)(e.uv >> 32);
      ev[at] = (unsigned)(e.uv & 0xffffffffu);
      ew[at] = e.w;
    }
    if (root[k] == (int)k) newid[k] = (int)(excl >> 31);
  }
};

__global__ void k_merge_final(const int* __restrict__ root, const int* __restrict__ newid, long long c, int* __restrict__ fin) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= c) return;
  fin[k] = newid[root[k]];
}

__global__ void k_relabel(int* __restrict__ label, const int* __restrict__ fin, long long n) {
  long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= n) return;
  label[s] = fin[label[s]];
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
// In-process stand-in for the two NCCL min-allreduces over V virtual shards
// (same two-phase protocol; used by the single-GPU shard-determinism tests).
__global__ void k_virtual_reduce(const EdgeKey* __restrict__ shard_keys, int shards, long long c, EdgeKey* __restrict__ best) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= c) return;
  unsigned long long w = ~0ull;
  for (int g = 0; g < shards; ++g) w = min(w, shard_keys[g * c + k].w);
  unsigned long long uv = ~0ull;
  for (int g = 0; g < shards; ++g) {
    EdgeKey e = shard_keys[g * c + k];
    if (e.w == w) uv = min(uv, e.uv);
  }
  EdgeKey r;
  r.w = w;
  r.uv = uv;
  best[k] = r;
}

// ------------------------------------------------------------ final output
__global__ void k_edge_uv_keys(const unsigned* __restrict__ eu, const unsigned* __restrict__ ev, long long ne,
                               unsigned long long* __restrict__ keys) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < ne) keys[i] = ((unsigned long long)eu[i] << 32) | ev[i];
}
__global__ void k_edge_w_keys(const unsigned long long* __restrict__ ew, const unsigned* __restrict__ order, long long ne,
                              unsigned long long* __restrict__ keys) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < ne) keys[i] = ew[order[i]];
}
__global__ void k_edge_emit(const unsigned* __restrict__ eu, const unsigned* __restrict__ ev,
                            const unsigned long long* __restrict__ ew, const unsigned* __restrict__ order, long long ne,
                            long long* __restrict__ edges, double* __restrict__ weights) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= ne) return;
  unsigned o = order[i];
  edges[2 * i] = eu[o];
  edges[2 * i + 1] = ev[o];
  weights[i] = __longlong_as_double((long long)ew[o]);
}

}  // namespace emst
