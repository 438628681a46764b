// wide.cuh -- traversal tree collapsed from the Karras binary LBVH to W = 2^L children.
//
// The binary tree stays the reference-exact structure (bvh.py numbering, exported
// for parity); the traversal runs on a wide copy of it: every binary node at a
// depth divisible by L becomes a wide node whose children are its descendants L
// levels down (leaves met earlier stay leaves).  A query then needs L times fewer
// dependent node fetches -- the traversal is latency bound (profiles/r01_*:
// long-scoreboard stalls dominate) -- and each fetch is one contiguous record
// loaded with 256-bit reads.  Results cannot change: any tree over the same
// points with conservative boxes and the same labels admits the same edges.
//
// Record (SoA so the W box tests vectorise): lo[D][W], hi[D][W], ref[W], label[W]
//   3D W=4: 128 B, 3D W=8: 256 B, 2D W=4: 96 B, 2D W=8: 192 B.
#pragma once
#include "common.cuh"
#include "scan.cuh"
#include "traverse.cuh"

namespace emst {

constexpr int kWideNone = (int)0x80000000;   // empty child slot

template <int D, int W>
struct __align__(32) WideNode {
  float lo[D][W];
  float hi[D][W];
  int ref[W];     // >= 0 wide node, < 0 leaf slot ~ref, kWideNone empty
  int label[W];   // per-round child component label, kMixed if mixed
};

// ---------------------------------------------------------------- build
// depth of every binary internal node by pointer jumping over node_parent
// (ping-pong buffers; ceil(log2(max depth)) launches).
__global__ void k_depth_init(const int* __restrict__ node_parent, long long m, int* __restrict__ anc, int* __restrict__ dep) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= m) return;
  anc[i] = i == 0 ? -1 : (node_parent[i] >> 1);
  dep[i] = i == 0 ? 0 : 1;
}
__global__ void k_depth_jump(const int* __restrict__ anc_in, const int* __restrict__ dep_in, long long m,
                             int* __restrict__ anc_out, int* __restrict__ dep_out) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= m) return;
  int a = anc_in[i];
  if (a < 0) { anc_out[i] = -1; dep_out[i] = dep_in[i]; return; }
  anc_out[i] = anc_in[a];
  dep_out[i] = dep_in[i] + dep_in[a];
}

template <int L>
struct KeptLoad {
  const int* dep;
  __device__ unsigned long long operator()(long long i) const { return dep[i] % L == 0 ? 1ull : 0ull; }
};
template <int L>
struct KeptStore {
  const int* dep;
  int* widx;
  __device__ void operator()(long long i, unsigned long long excl) const { widx[i] = dep[i] % L == 0 ? (int)excl : -1; }
};

__device__ __forceinline__ void binary_child_box(const Node3* nodes, int p, int side, float* lo, float* hi) {
  const float* f = reinterpret_cast<const float*>(&nodes[p]) + side * 6;
  lo[0] = f[0]; lo[1] = f[1]; lo[2] = f[2]; hi[0] = f[3]; hi[1] = f[4]; hi[2] = f[5];
}
__device__ __forceinline__ void binary_child_box(const Node2* nodes, int p, int side, float* lo, float* hi) {
  const float* f = reinterpret_cast<const float*>(&nodes[p]) + side * 4;
  lo[0] = f[0]; lo[1] = f[1]; hi[0] = f[2]; hi[1] = f[3]; lo[2] = hi[2] = 0.f;
}

template <int D, int L>
__global__ void k_collapse(const typename NodeOf<D>::type* __restrict__ nodes, const int2* __restrict__ range,
                           const int* __restrict__ widx, long long m, WideNode<D, (1 << L)>* __restrict__ wnodes,
                           int2* __restrict__ wrange) {
  constexpr int W = 1 << L;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int w = widx[i];
  if (w < 0) return;
  // frontier of (parent binary node, side, ref) expanded level by level
  int fp[W], fs[W], fr[W];
  int cnt = 2;
  const int4 r0 = nodes[i].ref;
  fp[0] = (int)i; fs[0] = 0; fr[0] = r0.x;
  fp[1] = (int)i; fs[1] = 1; fr[1] = r0.y;
#pragma unroll
  for (int lev = 1; lev < L; ++lev) {
    int np[W], ns[W], nr[W];
    int nc = 0;
#pragma unroll
    for (int k = 0; k < W; ++k) {
      if (k >= cnt) break;
      if (fr[k] < 0) { np[nc] = fp[k]; ns[nc] = fs[k]; nr[nc] = fr[k]; ++nc; continue; }
      const int4 rr = nodes[fr[k]].ref;
      np[nc] = fr[k]; ns[nc] = 0; nr[nc] = rr.x; ++nc;
      np[nc] = fr[k]; ns[nc] = 1; nr[nc] = rr.y; ++nc;
    }
#pragma unroll
    for (int k = 0; k < W; ++k) { if (k < nc) { fp[k] = np[k]; fs[k] = ns[k]; fr[k] = nr[k]; } }
    cnt = nc;
  }
  WideNode<D, W> out;
#pragma unroll
  for (int k = 0; k < W; ++k) {
    if (k < cnt) {
      float lo[3], hi[3];
      binary_child_box(nodes, fp[k], fs[k], lo, hi);
#pragma unroll
      for (int a = 0; a < D; ++a) { out.lo[a][k] = lo[a]; out.hi[a][k] = hi[a]; }
      const int c = fr[k];
      out.ref[k] = c < 0 ? c : widx[c];
      wrange[(long long)w * W + k] = c < 0 ? make_int2(~c, ~c) : range[c];
    } else {
#pragma unroll
      for (int a = 0; a < D; ++a) { out.lo[a][k] = __int_as_float(0x7f800000); out.hi[a][k] = -__int_as_float(0x7f800000); }
      out.ref[k] = kWideNone;
      wrange[(long long)w * W + k] = make_int2(0, 0);
    }
    out.label[k] = kMixed;
  }
  wnodes[w] = out;
}

// ----------------------------------------------------------- round labels
template <int D, int W>
__global__ void k_wide_labels(WideNode<D, W>* __restrict__ wnodes, const int2* __restrict__ wrange,
                              const int* __restrict__ bprefix, const int* __restrict__ label, long long mw) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;   // one thread per (node, child)
  if (t >= mw * W) return;
  const long long w = t / W;
  const int k = (int)(t % W);
  const int2 r = wrange[t];
  int l = kMixed;
  if (wnodes[w].ref[k] != kWideNone) l = bprefix[r.y] == bprefix[r.x] ? label[r.x] : kMixed;
  wnodes[w].label[k] = l;
}

// --------------------------------------------------------------- traversal
template <int D, int W>
__device__ __forceinline__ void load_wide(const WideNode<D, W>* p, WideNode<D, W>& r) {
  static_assert(sizeof(WideNode<D, W>) % 32 == 0, "wide node must be a multiple of 32 bytes");
  const float4* src = reinterpret_cast<const float4*>(p);
  float4* dst = reinterpret_cast<float4*>(&r);
#pragma unroll
  for (int j = 0; j < (int)(sizeof(WideNode<D, W>) / 16); j += 2) ldg256(src + j, dst[j], dst[j + 1]);
}

// Stack bound: each wide level can leave W-1 siblings behind; 96 binary levels
// cover any tree the 64-entry binary reference can traverse, so this capacity
// never overflows where the reference's would not.
template <int W>
struct WideStack { static constexpr int L = W == 8 ? 3 : (W == 4 ? 2 : 1); static constexpr int value = (W - 1) * ((96 + L - 1) / L) + 8; };

template <int D, int W, bool kSkip, bool kBounds>
__global__ void __launch_bounds__(kTraverseThreads, EMST_TRAV_MINB)
k_traverse_wide(const WideNode<D, W>* __restrict__ wnodes, const float4* __restrict__ spts,
                const unsigned* __restrict__ perm, const int* __restrict__ label, unsigned long long* ub,
                EdgeKey* __restrict__ best, long long q0, long long q1, const Box3* __restrict__ root_box,
                unsigned long long* __restrict__ evals_out, int* __restrict__ overflow,
                unsigned long long* __restrict__ work_counter) {
  const unsigned lane = lane_id();
  const unsigned lt = lanemask_lt_u32();
  const long long total = q1 - q0;
  float rlo[3], rhi[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) { rlo[k] = root_box->lo[k]; rhi[k] = root_box->hi[k]; }

  long long pool_next = 0, pool_end = 0;
  bool exhausted = false;
  long long s = -1;
  float q[3] = {0.f, 0.f, 0.f};
  unsigned qp = 0;
  int comp = 0;
  double radius = 0.0;
  float r2 = 0.f;
  unsigned long long best_w = ~0ull, best_uv = ~0ull;
  constexpr int kCap = WideStack<W>::value;
  int stack_node[kCap];
  float stack_lb[kCap];
  int top = 0;
  int since_refresh = 0;
  unsigned long long evals = 0;

  for (;;) {
    const unsigned idle = __ballot_sync(0xffffffffu, s < 0);
    const int n_idle = __popc(idle);
    if (n_idle == 32 && exhausted) break;
    if (n_idle >= kRefillIdle || n_idle == 32) {
      if (pool_next >= pool_end && !exhausted) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(work_counter, (unsigned long long)kTraverseChunk);
        base = __shfl_sync(0xffffffffu, base, 0);
        if ((long long)base >= total) {
          exhausted = true;
        } else {
          pool_next = (long long)base;
          pool_end = min((long long)base + kTraverseChunk, total);
        }
      }
      if (pool_next < pool_end) {
        const unsigned rank = __popc(idle & lt);
        const long long mine = pool_next + (long long)rank;
        const bool take = s < 0 && mine < pool_end;
        pool_next = min(pool_end, pool_next + (long long)n_idle);
        if (take) {
          s = mine;
          const long long slot = q0 + s;
          const float4 qv = spts[slot];
          q[0] = qv.x; q[1] = qv.y; q[2] = qv.z;
          qp = __float_as_uint(qv.w);
          comp = label[slot];
          radius = kBounds ? bits_to_radius(__ldcg(&ub[comp])) : __longlong_as_double(0x7ff0000000000000ll);
          r2 = prune_r2(radius);
          best_w = ~0ull;
          best_uv = ~0ull;
          stack_node[0] = 0;
          stack_lb[0] = box_lb2<D>(q, rlo, rhi);
          top = 1;
          since_refresh = 0;
        }
      }
    }
    if (s < 0) continue;

    --top;
    const float plb = stack_lb[top];
    if (kBounds && ++since_refresh >= kRadiusRefresh) {
      since_refresh = 0;
      const double shared = bits_to_radius(__ldcg(&ub[comp]));
      if (shared < radius) { radius = shared; r2 = prune_r2(shared); }
    }
    if (plb <= r2) {
      WideNode<D, W> rec;
      load_wide<D, W>(wnodes + stack_node[top], rec);
      float key[W];
      int cid[W];
#pragma unroll
      for (int k = 0; k < W; ++k) {
        const int c = rec.ref[k];
        float lo[3], hi[3];
#pragma unroll
        for (int a = 0; a < D; ++a) { lo[a] = rec.lo[a][k]; hi[a] = rec.hi[a][k]; }
        const float lb = box_lb2<D>(q, lo, hi);
        const bool same = rec.label[k] == comp && (c < 0 || kSkip);
        bool want = c != kWideNone && !same && lb <= r2;
        if (want && c < 0) {
          want = false;
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
              if (w < radius) {
                radius = w;
                r2 = prune_r2(w);
                if (kBounds) atomicMin(&ub[comp], wb);
              }
            }
          }
        }
        key[k] = want ? lb : __int_as_float(0x7f800000);
        cid[k] = c;
      }
      // ascending sort of the (<= W) wanted children by lower bound; unwanted sink (+inf)
#pragma unroll
      for (int a = 0; a < W; ++a) {
#pragma unroll
        for (int b = 0; b + 1 < W - a; ++b) {
          if (key[b + 1] < key[b]) {
            const float tk = key[b]; key[b] = key[b + 1]; key[b + 1] = tk;
            const int tc = cid[b]; cid[b] = cid[b + 1]; cid[b + 1] = tc;
          }
        }
      }
      int np = 0;
#pragma unroll
      for (int k = 0; k < W; ++k) np += key[k] != __int_as_float(0x7f800000);
      if (top + np > kCap) {
        atomicOr(overflow, 1);
        top = 0;
      } else {
        // farthest first so the nearest child is popped next
#pragma unroll
        for (int k = W - 1; k >= 0; --k) {
          if (k < np) {
            stack_node[top] = cid[k];
            stack_lb[top] = key[k];
            ++top;
          }
        }
      }
    }
    if (top == 0) {
      if (best_uv != ~0ull) atomic_min_key(&best[comp], best_w, best_uv);
      s = -1;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) evals += __shfl_xor_sync(0xffffffffu, evals, o);
  if (lane == 0 && evals) atomicAdd(evals_out, evals);
}

}  // namespace emst
