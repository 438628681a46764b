// core.cuh -- core distances for the mutual-reachability metric (reference
// metric.py:128-234): core(p) = the distance from p to its k_pts-th nearest
// neighbour counting p itself, i.e. the (k_pts - 1)-th smallest exact f64
// distance from p to the OTHER points (duplicates count, at distance 0).
//
// k_core is the climb traversal of traverse.cuh (a query starts at its own
// leaf and climbs, exploring sibling subtrees nearest-first; its own leaf is
// never visited) with a bounded max-heap of the kc = k_pts - 1 smallest
// distances per query.  The pruning radius is the heap top (prune_r2 slack,
// strict f32 lower bounds), so a pruned box only holds points strictly farther
// than the current kc-th distance and cannot change its value -- ties do not
// matter for a value.  Only the value is kept (no indices).  The heap lives in
// shared memory laid out [entry][thread], or for large k_pts in a global
// scratch area [entry][lane of the grid] (same code through a generic pointer).
#pragma once
#include "traverse.cuh"

namespace emst {

constexpr int kCoreThreads = 128;
constexpr int kCoreChunk = 64;
constexpr int kCoreSmemStack = 8;

template <int D>
__global__ void __launch_bounds__(kCoreThreads)
k_core(const typename NodeOf<D>::type* __restrict__ nodes, const float4* __restrict__ spts, long long q0, long long q1,
       int kc, double* heap_global, double* __restrict__ core_out, unsigned long long* __restrict__ counters,
       int* __restrict__ overflow, unsigned long long* __restrict__ work_counter, const int2* __restrict__ up,
       const int* __restrict__ leaf_parent, const Scene* __restrict__ scene_ptr) {
  extern __shared__ double s_heap[];   // [kc][kCoreThreads] unless heap_global
  __shared__ int2 s_stk[kCoreSmemStack][kCoreThreads];
  int2 deep[kStackCapacity - kCoreSmemStack];
  const unsigned lane = lane_id();
  const unsigned lt = lanemask_lt_u32();
  const int tid = threadIdx.x;
  const int total = (int)(q1 - q0);
  const Scene sc = *scene_ptr;
  // entry j of this lane's heap is h[j * hs]
  double* h = heap_global ? heap_global + (long long)blockIdx.x * blockDim.x + tid : s_heap + tid;
  const long long hs = heap_global ? (long long)gridDim.x * blockDim.x : (long long)kCoreThreads;

  int pool_next = 0, pool_end = 0;
  bool exhausted = false;
  int s = -1;
  float q[3] = {0.f, 0.f, 0.f};
  int size = 0;
  float r2 = 0.f;
  int top = 0, climb = -1, path_side = 0, prefix = -1;
  float prefix_r2 = 0.f;
  unsigned evals = 0, visits = 0;

  auto stk_get = [&](int i) -> int2 { return i < kCoreSmemStack ? s_stk[i][tid] : deep[i - kCoreSmemStack]; };
  auto stk_put = [&](int i, int node, float lb) {
    const int2 e = make_int2(node, __float_as_int(lb));
    if (i < kCoreSmemStack) s_stk[i][tid] = e; else deep[i - kCoreSmemStack] = e;
  };
  // bounded max-heap of the kc smallest distances
  auto offer = [&](double d) {
    if (size < kc) {
      int i = size++;
      while (i > 0) {
        const int p = (i - 1) >> 1;
        const double hp = h[p * hs];
        if (!(hp < d)) break;
        h[i * hs] = hp;
        i = p;
      }
      h[i * hs] = d;
    } else {
      if (!(d < h[0])) return;
      int i = 0;
      for (;;) {
        const int l = 2 * i + 1;
        if (l >= kc) break;
        int b = l;
        double hb = h[l * hs];
        if (l + 1 < kc) {
          const double hr = h[(l + 1) * hs];
          if (hr > hb) { b = l + 1; hb = hr; }
        }
        if (!(hb > d)) break;
        h[i * hs] = hb;
        i = b;
      }
      h[i * hs] = d;
    }
    if (size == kc) r2 = prune_r2(h[0]);
  };

  for (;;) {
    const unsigned idle = __ballot_sync(0xffffffffu, s < 0);
    const int n_idle = __popc(idle);
    if (n_idle == 32 && exhausted) break;
    if (n_idle >= 16) {
      if (pool_next >= pool_end && !exhausted) {
        unsigned long long base = 0;
        if (lane == 0) {
          base = atomicAdd(work_counter, (unsigned long long)kCoreChunk);
#if EMST_TRAV_PREFETCH
          const long long a = q0 + (long long)base + kTravPrefetch;   // (as in k_traverse)
          if (a + kCoreChunk < q1) {
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;"
                         :: "l"(nodes + a), "r"((unsigned)(kCoreChunk * sizeof(*nodes))) : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;"
                         :: "l"(spts + a), "r"((unsigned)(kCoreChunk * sizeof(float4))) : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;"
                         :: "l"(up + a), "r"((unsigned)(kCoreChunk * sizeof(int2))) : "memory");
          }
#endif
        }
        base = __shfl_sync(0xffffffffu, base, 0);
        if ((long long)base >= total) {
          exhausted = true;
        } else {
          pool_next = (int)base;
          pool_end = min((int)base + kCoreChunk, total);
        }
      }
      if (pool_next < pool_end) {
        const int rank = __popc(idle & lt);
        const int mine = pool_next + rank;
        const bool take = s < 0 && mine < pool_end;
        pool_next = min(pool_end, pool_next + n_idle);
        if (take) {
          s = mine;
          const float4 qv = __ldg(spts + q0 + s);
          q[0] = qv.x; q[1] = qv.y; q[2] = qv.z;
          size = 0;
          r2 = __int_as_float(0x7f800000);
          top = 0;
          const int link = __ldg(leaf_parent + q0 + s);
          climb = link >> 1;
          path_side = link & 1;
          prefix = -1;
          prefix_r2 = __int_as_float(0x7f800000);
        }
      }
    }
    if (s < 0) continue;

    int2 e = make_int2(-1, 0);
    while (top > 0) {
      e = stk_get(top - 1);
      if (__int_as_float(e.y) <= r2) break;
      --top;
      e.x = -1;
    }
    int node;
    unsigned sides;
    const bool climbing = top == 0;
    if (!climbing) {
      --top;
      node = e.x;
      sides = 3u;
    } else {
      node = climb;
      sides = 2u >> path_side;
    }
    if (node >= 0) {
      ++visits;
      const auto rec = load_node(nodes + node);
      int2 u = make_int2(-1, 0);
      if (climbing) u = __ldg(up + node);
      float lbs[2];
      node_lb2(rec, q, lbs[0], lbs[1]);
      bool want[2] = {false, false};
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        if (!((sides >> side) & 1u) || lbs[side] > r2) continue;
        const int c = side ? rec.ref.y : rec.ref.x;
        if (c >= 0) {
          want[side] = true;
        } else {
          float lo[3], hi[3];
          child_box<D>(rec, side, lo, hi);
          ++evals;
          offer(exact_dist<D>(q, lo));
        }
      }
      const bool want0 = want[0] && lbs[0] <= r2, want1 = want[1] && lbs[1] <= r2;
      const int np = (int)want0 + (int)want1;
      if (top + np > kStackCapacity) {
        atomicOr(overflow, 1);
        top = 0;
        climb = -1;
      } else if (np == 2) {
        const bool near1 = lbs[1] < lbs[0];
        stk_put(top, near1 ? rec.ref.x : rec.ref.y, near1 ? lbs[0] : lbs[1]);
        stk_put(top + 1, near1 ? rec.ref.y : rec.ref.x, near1 ? lbs[1] : lbs[0]);
        top += 2;
      } else if (np == 1) {
        stk_put(top, want0 ? rec.ref.x : rec.ref.y, want0 ? lbs[0] : lbs[1]);
        ++top;
      }
      if (climbing && climb >= 0) {
        // (as in k_traverse: a prefix for a larger search radius stays valid)
        if (u.y > prefix && r2 <= 0.25f * prefix_r2) {
          prefix = ball_prefix<D>(q, (double)__fsqrt_ru(r2), sc);
          prefix_r2 = r2;
        }
        if (u.y <= prefix || u.x < 0) {
          climb = -1;
        } else {
          climb = u.x >> 1;
          path_side = u.x & 1;
        }
      }
    }
    if (top == 0 && climb < 0) {
      core_out[q0 + s] = h[0];   // (kc <= n - 1 points are always found)
      s = -1;
    }
  }
  unsigned long long ev64 = evals, vi64 = visits;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ev64 += __shfl_xor_sync(0xffffffffu, ev64, o);
    vi64 += __shfl_xor_sync(0xffffffffu, vi64, o);
  }
  if (lane == 0) {
    if (ev64) atomicAdd(counters, ev64);
    if (vi64) atomicAdd(counters + 5, vi64);
  }
}

// slot order <-> original order for per-point f64 tables
__global__ void k_gather_by_perm(const double* __restrict__ by_point, const unsigned* __restrict__ perm, long long n,
                                 double* __restrict__ by_slot) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s < n) by_slot[s] = by_point[perm[s]];
}
__global__ void k_scatter_by_perm(const double* __restrict__ by_slot, const unsigned* __restrict__ perm, long long n,
                                  double* __restrict__ by_point) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s < n) by_point[perm[s]] = by_slot[s];
}

}  // namespace emst
