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
      atomicMin(&ub[la], bits);
      atomicMin(&ub[lb], bits);
    }
    return 1ull;
  }
};
struct RoundScanStore {
  int* bprefix;
  __device__ void operator()(long long i, unsigned long long excl) const { bprefix[i] = (int)excl; }
};

// ------------------------------------------------------------- node labels
template <class Node>
__global__ void k_node_labels(Node* __restrict__ nodes, const int2* __restrict__ range, const int* __restrict__ bprefix,
                              const int* __restrict__ label, long long m) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= m) return;
  int2 r = range[i];
  int lref = nodes[i].ref.x;
  int gamma = lref >= 0 ? lref : ~lref;
  int bl = bprefix[r.x], bg = bprefix[gamma], bg1 = bprefix[gamma + 1], bh = bprefix[r.y];
  int ll = bg == bl ? label[r.x] : kMixed;
  int rl = bh == bg1 ? label[r.y] : kMixed;
  *reinterpret_cast<int2*>(&nodes[i].ref.z) = make_int2(ll, rl);
}

// ---------------------------------------------------------------- traversal
template <int D>
__device__ __forceinline__ void child_box(const Node3& rec, int side, float* lo, float* hi) {
  if (side == 0) {
    lo[0] = rec.a.x; lo[1] = rec.a.y; lo[2] = rec.a.z; hi[0] = rec.a.w; hi[1] = rec.b.x; hi[2] = rec.b.y;
  } else {
    lo[0] = rec.b.z; lo[1] = rec.b.w; lo[2] = rec.c.x; hi[0] = rec.c.y; hi[1] = rec.c.z; hi[2] = rec.c.w;
  }
}
template <int D>
__device__ __forceinline__ void child_box(const Node2& rec, int side, float* lo, float* hi) {
  const float4& v = side == 0 ? rec.a : rec.b;
  lo[0] = v.x; lo[1] = v.y; hi[0] = v.z; hi[1] = v.w; lo[2] = hi[2] = 0.f;
}

__device__ __forceinline__ Node3 load_node(const Node3* p) {
  const float4* f = reinterpret_cast<const float4*>(p);
  Node3 r;
  r.a = __ldg(f);
  r.b = __ldg(f + 1);
  r.c = __ldg(f + 2);
  r.ref = __ldg(reinterpret_cast<const int4*>(f + 3));
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

constexpr int kTraverseThreads = 256;

template <int D, bool kSkip, bool kBounds>
__global__ void __launch_bounds__(kTraverseThreads)
k_traverse(const typename NodeOf<D>::type* __restrict__ nodes, const float4* __restrict__ spts,
           const unsigned* __restrict__ perm, const int* __restrict__ label,
           const unsigned long long* __restrict__ ub, EdgeKey* __restrict__ best, long long q0, long long q1,
           const Box3* __restrict__ root_box, unsigned long long* __restrict__ evals_out, int* __restrict__ overflow) {
  const long long s = q0 + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  unsigned long long evals = 0;
  if (s < q1) {
    const float4 qv = spts[s];
    const float q[3] = {qv.x, qv.y, qv.z};
    const unsigned qp = __float_as_uint(qv.w);
    const int comp = label[s];
    double radius = kBounds ? bits_to_radius(ub[comp]) : __longlong_as_double(0x7ff0000000000000ll);
    float r2 = prune_r2(radius);
    unsigned long long best_w = ~0ull, best_uv = ~0ull;

    int stack_node[kStackCapacity];
    float stack_lb[kStackCapacity];
    stack_node[0] = 0;
    stack_lb[0] = box_lb2<D>(q, root_box->lo, root_box->hi);
    int top = 1;
    while (top > 0) {
      --top;
      if (stack_lb[top] > r2) continue;
      const auto rec = load_node(nodes + stack_node[top]);
      int push_node[2];
      float push_lb[2];
      int np = 0;
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        const int c = side ? rec.ref.y : rec.ref.x;
        const int cl = side ? rec.ref.w : rec.ref.z;
        float lo[3], hi[3];
        child_box<D>(rec, side, lo, hi);
        if (c < 0) {
          if (cl == comp) continue;
          ++evals;
          const double w = exact_dist<D>(q, lo);
          if (w <= radius) {
            const unsigned p = __ldg(perm + (~c));
            const unsigned long long u = qp < p ? qp : p, v = qp < p ? p : qp;
            const unsigned long long uv = (u << 32) | v;
            const unsigned long long wb = (unsigned long long)__double_as_longlong(w);
            if (key_less(wb, uv, best_w, best_uv)) {
              best_w = wb;
              best_uv = uv;
              radius = w;
              r2 = prune_r2(w);
            }
          }
        } else {
          if (kSkip && cl == comp) continue;
          const float lb = box_lb2<D>(q, lo, hi);
          if (lb <= r2) {
            push_node[np] = c;
            push_lb[np] = lb;
            ++np;
          }
        }
      }
      if (np == 2) {
        if (top + 2 > kStackCapacity) { atomicOr(overflow, 1); break; }
        // nearer child on top (popped first); ties keep the left child there
        const int near = push_lb[1] < push_lb[0] ? 1 : 0;
        stack_node[top] = push_node[1 - near];
        stack_lb[top] = push_lb[1 - near];
        stack_node[top + 1] = push_node[near];
        stack_lb[top + 1] = push_lb[near];
        top += 2;
      } else if (np == 1) {
        if (top + 1 > kStackCapacity) { atomicOr(overflow, 1); break; }
        stack_node[top] = push_node[0];
        stack_lb[top] = push_lb[0];
        ++top;
      }
    }
    if (best_uv != ~0ull) atomic_min_key(&best[comp], best_w, best_uv);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) evals += __shfl_xor_sync(0xffffffffu, evals, o);
  if (lane_id() == 0 && evals) atomicAdd(evals_out, evals);
}

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
