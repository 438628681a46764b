// build.cuh -- LBVH construction kernels (reference: geometry.py, bvh.py:305-340).
//
//   k_scene         bounds + finiteness in one read of the points; the last block
//                   folds the per-block partials and derives lo / 1/extent in f64
//                   (geometry.py:36-71, 102-105, 201-206)
//   k_morton        bit-exact quantise + interleave (geometry.py:143-227)
//   (radix sort)    stable Z-order permutation (bvh.py:317)
//   k_gather        float4 points in slot order, perm / iperm as u32
//   k_karras        radix-tree topology, node numbering identical to the
//                   reference's _build_topology (bvh.py:112-201)
//   k_refit         bottom-up boxes by atomic-arrival climb: the second thread to
//                   reach a node combines its children (replaces the serial level
//                   schedule of bvh.py:204-264, 293-302)
#pragma once
#include "common.cuh"

namespace emst {

constexpr int kSceneThreads = 256;

template <int D>
__global__ void __launch_bounds__(kSceneThreads)
k_scene(const float* __restrict__ pts, long long n, float* __restrict__ part_lo, float* __restrict__ part_hi,
        long long* __restrict__ part_bad, Scene* __restrict__ scene) {
  float lo[D], hi[D];
#pragma unroll
  for (int k = 0; k < D; ++k) { lo[k] = __int_as_float(0x7f800000); hi[k] = -__int_as_float(0x7f800000); }
  long long bad = 0x7fffffffffffffffll;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  // 16-byte aligned input (the usual case): 4 points per step as D float4 loads
  const bool vec = (reinterpret_cast<unsigned long long>(pts) & 15ull) == 0;
  const long long nv = vec ? n / 4 : 0;
  for (long long t = t0; t < nv; t += stride) {
    const float4* v = reinterpret_cast<const float4*>(pts) + t * D;
    float f[4 * D];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const float4 x = __ldg(v + j);
      f[4 * j] = x.x; f[4 * j + 1] = x.y; f[4 * j + 2] = x.z; f[4 * j + 3] = x.w;
    }
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      bool fin = true;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const float x = f[p * D + k];
        fin &= isfinite(x);
        lo[k] = fminf(lo[k], x);
        hi[k] = fmaxf(hi[k], x);
      }
      if (!fin && 4 * t + p < bad) bad = 4 * t + p;
    }
  }
  for (long long i = nv * 4 + t0; i < n; i += stride) {
    bool fin = true;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      float x = pts[i * D + k];
      fin &= isfinite(x);
      lo[k] = fminf(lo[k], x);
      hi[k] = fmaxf(hi[k], x);
    }
    if (!fin && i < bad) bad = i;
  }
  __shared__ float s_lo[D][kSceneThreads / 32], s_hi[D][kSceneThreads / 32];
  __shared__ long long s_bad[kSceneThreads / 32];
  __shared__ bool s_last;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      lo[k] = fminf(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
      hi[k] = fmaxf(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
    }
    long long b = __shfl_xor_sync(0xffffffffu, bad, o);
    bad = b < bad ? b : bad;
  }
  const int w = threadIdx.x >> 5;
  if (lane_id() == 0) {
#pragma unroll
    for (int k = 0; k < D; ++k) { s_lo[k][w] = lo[k]; s_hi[k][w] = hi[k]; }
    s_bad[w] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int j = 1; j < kSceneThreads / 32; ++j) {
#pragma unroll
      for (int k = 0; k < D; ++k) { lo[k] = fminf(lo[k], s_lo[k][j]); hi[k] = fmaxf(hi[k], s_hi[k][j]); }
      bad = s_bad[j] < bad ? s_bad[j] : bad;
    }
#pragma unroll
    for (int k = 0; k < D; ++k) { part_lo[blockIdx.x * D + k] = lo[k]; part_hi[blockIdx.x * D + k] = hi[k]; }
    part_bad[blockIdx.x] = bad;
    __threadfence();
    unsigned done = atomicAdd(&scene->blocks_done, 1u);
    s_last = done == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  // the last block folds the per-block partials, all its threads at once
  __threadfence();
  for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      lo[k] = fminf(lo[k], __ldcg(&part_lo[b * D + k]));
      hi[k] = fmaxf(hi[k], __ldcg(&part_hi[b * D + k]));
    }
    long long pb = __ldcg(&part_bad[b]);
    bad = pb < bad ? pb : bad;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      lo[k] = fminf(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
      hi[k] = fmaxf(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
    }
    long long bb = __shfl_xor_sync(0xffffffffu, bad, o);
    bad = bb < bad ? bb : bad;
  }
  __syncthreads();   // (s_lo / s_hi / s_bad are reused)
  if (lane_id() == 0) {
#pragma unroll
    for (int k = 0; k < D; ++k) { s_lo[k][w] = lo[k]; s_hi[k][w] = hi[k]; }
    s_bad[w] = bad;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int j = 1; j < kSceneThreads / 32; ++j) {
#pragma unroll
    for (int k = 0; k < D; ++k) { lo[k] = fminf(lo[k], s_lo[k][j]); hi[k] = fmaxf(hi[k], s_hi[k][j]); }
    bad = s_bad[j] < bad ? s_bad[j] : bad;
  }
  scene->bad_row = bad;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    float l = k < D ? lo[k] : 0.f, h = k < D ? hi[k] : 0.f;
    scene->flo[k] = l;
    scene->fhi[k] = h;
    double ext = __dsub_rn((double)h, (double)l);
    scene->lo[k] = (double)l;
    scene->inv[k] = ext > 0.0 ? __drcp_rn(ext) : 0.0;   // IEEE 1/ext (geometry.py:205)
    scene->cellw[k] = ext > 0.0 ? __drcp_rn(scene->inv[k] * (D == 3 ? 2097152.0 : 2147483648.0)) : 0.0;
  }
  scene->blocks_done = 0;
}

template <int D>
__global__ void k_morton(const float* __restrict__ pts, long long n, const Scene* __restrict__ scene,
                         unsigned long long* __restrict__ codes) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (D == 3) {
    const double scale = 2097152.0;   // 2^21
    unsigned long long cx = lattice_cell(pts[i * 3 + 0], scene->lo[0], scene->inv[0], scale);
    unsigned long long cy = lattice_cell(pts[i * 3 + 1], scene->lo[1], scene->inv[1], scale);
    unsigned long long cz = lattice_cell(pts[i * 3 + 2], scene->lo[2], scene->inv[2], scale);
    codes[i] = (spread_bits3(cx) << 2) | (spread_bits3(cy) << 1) | spread_bits3(cz);
  } else {
    const double scale = 2147483648.0;   // 2^31
    unsigned long long cx = lattice_cell(pts[i * 2 + 0], scene->lo[0], scene->inv[0], scale);
    unsigned long long cy = lattice_cell(pts[i * 2 + 1], scene->lo[1], scene->inv[1], scale);
    codes[i] = (spread_bits2(cx) << 1) | spread_bits2(cy);
  }
}

// Slot-order points: kGatherPer slots per thread so that many independent
// random point reads are in flight per thread (the reads follow the Morton
// permutation and are latency-bound); also writes perm and its inverse.
constexpr int kGatherThreads = 256;
constexpr int kGatherPer = 4;

template <int D>
__global__ void __launch_bounds__(kGatherThreads)
k_gather(const float* __restrict__ pts, long long n, const unsigned* __restrict__ sorted_idx,
         unsigned* __restrict__ perm, float4* __restrict__ spts, unsigned* __restrict__ iperm,
         const Scene* __restrict__ scene, unsigned long long* __restrict__ codes) {
  const long long base = (long long)blockIdx.x * (kGatherThreads * kGatherPer) + threadIdx.x;
  unsigned p[kGatherPer];
  float4 v[kGatherPer];
#pragma unroll
  for (int j = 0; j < kGatherPer; ++j) {
    const long long s = base + j * kGatherThreads;
    p[j] = s < n ? sorted_idx[s] : 0u;
  }
#pragma unroll
  for (int j = 0; j < kGatherPer; ++j) {
    const long long s = base + j * kGatherThreads;
    if (s < n) {
      v[j].x = pts[(long long)p[j] * D + 0];
      v[j].y = pts[(long long)p[j] * D + 1];
      v[j].z = D == 3 ? pts[(long long)p[j] * D + 2] : 0.f;
      v[j].w = __uint_as_float(p[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < kGatherPer; ++j) {
    const long long s = base + j * kGatherThreads;
    if (s < n) {
      spts[s] = v[j];
      perm[s] = p[j];
      if (iperm) iperm[p[j]] = (unsigned)s;
      // the sorted Morton codes, recomputed from the gathered point (the sort's
      // last pass writes only the permutation): k_morton's formula, bit for bit
      if (codes) {
        if (D == 3)
          codes[s] = (spread_bits3(lattice_cell(v[j].x, scene->lo[0], scene->inv[0], 2097152.0)) << 2) |
                     (spread_bits3(lattice_cell(v[j].y, scene->lo[1], scene->inv[1], 2097152.0)) << 1) |
                     spread_bits3(lattice_cell(v[j].z, scene->lo[2], scene->inv[2], 2097152.0));
        else
          codes[s] = (spread_bits2(lattice_cell(v[j].x, scene->lo[0], scene->inv[0], 2147483648.0)) << 1) |
                     spread_bits2(lattice_cell(v[j].y, scene->lo[1], scene->inv[1], 2147483648.0));
      }
    }
  }
}

// iperm[perm[s]] = s for the targets p in [lo, hi): the random 4-byte scatter
// runs over one part of iperm at a time, small enough to stay in L2 until its
// sectors are complete (one pass over all 148 MB at 37M scatters straight to DRAM
// and costs 1.3 ms of partial-sector writes).  perm is read once per part.
__global__ void __launch_bounds__(256) k_inverse_perm(const unsigned* __restrict__ perm, long long n, unsigned lo,
                                                      unsigned hi, unsigned* __restrict__ iperm) {
  const long long n4 = n >> 2;
  const uint4* p4 = reinterpret_cast<const uint4*>(perm);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const uint4 v = __ldg(p4 + i);
    const unsigned s = (unsigned)(i << 2);
    if (v.x - lo < hi - lo) iperm[v.x] = s;
    if (v.y - lo < hi - lo) iperm[v.y] = s + 1;
    if (v.z - lo < hi - lo) iperm[v.z] = s + 2;
    if (v.w - lo < hi - lo) iperm[v.w] = s + 3;
  }
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    const long long s = (n4 << 2) + threadIdx.x;
    const unsigned v = perm[s];
    if (v - lo < hi - lo) iperm[v] = (unsigned)s;
  }
}

// Common-prefix length of augmented keys (code, slot); -1 out of range (bvh.py:138-149).
__device__ __forceinline__ int aug_prefix(const unsigned long long* __restrict__ c, long long n, long long i, long long j) {
  if (j < 0 || j >= n) return -1;
  unsigned long long a = c[i], b = c[j];
  if (a != b) return __clzll((long long)(a ^ b));
  return 64 + __clzll((long long)((unsigned long long)i ^ (unsigned long long)j));
}

// node ref packing: internal i -> i, leaf slot s -> ~s
__device__ __forceinline__ int leaf_ref(long long s) { return ~(int)s; }

template <class Node>
__global__ void k_karras(const unsigned long long* __restrict__ sc, long long n, Node* __restrict__ nodes,
                         int2* __restrict__ range, int* __restrict__ node_parent, int* __restrict__ leaf_parent,
                         int* __restrict__ node_delta) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long m = n - 1;
  if (i >= m) return;
  const int dir = aug_prefix(sc, n, i, i + 1) > aug_prefix(sc, n, i, i - 1) ? 1 : -1;
  const int floor_len = aug_prefix(sc, n, i, i - dir);
  long long span = 2;
  while (aug_prefix(sc, n, i, i + span * dir) > floor_len) span <<= 1;
  long long len = 0;
  for (long long step = span >> 1; step >= 1; step >>= 1)
    if (aug_prefix(sc, n, i, i + (len + step) * dir) > floor_len) len += step;
  const long long j = i + len * dir;
  const int node_len = aug_prefix(sc, n, i, j);
  long long s = 0, step = len;
  while (step > 1) {
    step = (step + 1) >> 1;
    if (aug_prefix(sc, n, i, i + (s + step) * dir) > node_len) s += step;
  }
  const long long gamma = i + s * dir + (dir < 0 ? -1 : 0);
  const long long lo = i < j ? i : j, hi = i < j ? j : i;
  int lref, rref;
  if (lo == gamma) { lref = leaf_ref(gamma); leaf_parent[gamma] = (int)(i << 1); }
  else { lref = (int)gamma; node_parent[gamma] = (int)(i << 1); }
  if (hi == gamma + 1) { rref = leaf_ref(gamma + 1); leaf_parent[gamma + 1] = (int)((i << 1) | 1); }
  else { rref = (int)(gamma + 1); node_parent[gamma + 1] = (int)((i << 1) | 1); }
  nodes[i].ref = make_int4(lref, rref, kMixed, kMixed);
  range[i] = make_int2((int)lo, (int)hi);
  node_delta[i] = node_len;
  if (i == 0) node_parent[0] = -1;
}

// (parent link, prefix length) per internal node: one 8-byte load per climb step
__global__ void k_pack_up(const int* __restrict__ node_parent, const int* __restrict__ node_delta, long long m,
                          int2* __restrict__ up) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < m) up[i] = make_int2(node_parent[i], node_delta[i]);
}

// --- child box slots inside a node record
// (child coordinates interleaved: lo[k] at 2k + side, hi[k] at 2D + 2k + side)
__device__ __forceinline__ void put_child_box(Node3* nodes, int node, int side, const float* lo, const float* hi) {
  float* f = reinterpret_cast<float*>(&nodes[node]) + side;
  f[0] = lo[0]; f[2] = lo[1]; f[4] = lo[2]; f[6] = hi[0]; f[8] = hi[1]; f[10] = hi[2];
}
__device__ __forceinline__ void put_child_box(Node2* nodes, int node, int side, const float* lo, const float* hi) {
  float* f = reinterpret_cast<float*>(&nodes[node]) + side;
  f[0] = lo[0]; f[2] = lo[1]; f[4] = hi[0]; f[6] = hi[1];
}
// L2-coherent read of both child boxes (written by other threads of this launch)
__device__ __forceinline__ void get_union_box(const Node3* nodes, int node, float* lo, float* hi) {
  const float4* p = reinterpret_cast<const float4*>(&nodes[node]);
  float4 a = __ldcg(p), b = __ldcg(p + 1), c = __ldcg(p + 2);
  lo[0] = fminf(a.x, a.y); lo[1] = fminf(a.z, a.w); lo[2] = fminf(b.x, b.y);
  hi[0] = fmaxf(b.z, b.w); hi[1] = fmaxf(c.x, c.y); hi[2] = fmaxf(c.z, c.w);
}
__device__ __forceinline__ void get_union_box(const Node2* nodes, int node, float* lo, float* hi) {
  const float4* p = reinterpret_cast<const float4*>(&nodes[node]);
  float4 a = __ldcg(p), b = __ldcg(p + 1);
  lo[0] = fminf(a.x, a.y); lo[1] = fminf(a.z, a.w);
  hi[0] = fmaxf(b.x, b.y); hi[1] = fmaxf(b.z, b.w);
  lo[2] = hi[2] = 0.f;
}

// both child boxes of a node at once (sides a = left, b = right), vector stores
__device__ __forceinline__ void put_node_boxes(Node3* nodes, int node, const float* alo, const float* ahi,
                                               const float* blo, const float* bhi) {
  float4* p = reinterpret_cast<float4*>(&nodes[node]);
  p[0] = make_float4(alo[0], blo[0], alo[1], blo[1]);
  p[1] = make_float4(alo[2], blo[2], ahi[0], bhi[0]);
  p[2] = make_float4(ahi[1], bhi[1], ahi[2], bhi[2]);
}
__device__ __forceinline__ void put_node_boxes(Node2* nodes, int node, const float* alo, const float* ahi,
                                               const float* blo, const float* bhi) {
  float4* p = reinterpret_cast<float4*>(&nodes[node]);
  p[0] = make_float4(alo[0], blo[0], alo[1], blo[1]);
  p[1] = make_float4(ahi[0], bhi[0], ahi[1], bhi[1]);
}

#ifndef EMST_REFIT_THREADS
#define EMST_REFIT_THREADS 256
#endif
constexpr int kRefitThreads = EMST_REFIT_THREADS;

// Bottom-up boxes in two kernels.  k_refit: a block owns the kRefitThreads
// consecutive slots [B, E) and the internal nodes of the same indices.  A node
// whose slot range lies inside the block (Karras: its index is then in [B, E)
// too) gets both child boxes at once from a sparse table of the block's points
// in shared memory (level l holds the box of slots [t, t + 2^l)); any range is
// the union of two overlapping power-of-two windows.  No arrival protocol, no
// divergence, no dependent global reads.  The roots of the block's subtrees
// (a leaf or an inside node whose parent straddles the block edge) put their
// box into the parent's record and count an acq_rel arrival; the second
// arrival lists the parent for k_refit_up, which climbs the upper tree.
constexpr int kRefitLevels = 9;   // 2^8 = kRefitThreads: a node can span the whole block
template <int D>
constexpr size_t refit_smem() { return (size_t)kRefitLevels * kRefitThreads * 6 * sizeof(float); }

// table layout [level][coordinate][slot] (lo 0..D-1, hi D..2D-1): conflict-free per coordinate
__device__ __forceinline__ int refit_at(int l, int k, int t) { return (l * 6 + k) * kRefitThreads + t; }

template <int D>
__device__ __forceinline__ void refit_query(const float* tab, int a, int b, float* lo, float* hi) {
  // box of block-relative slots [a, b] (inclusive)
  const int len = b - a + 1;
  const int l = 31 - __clz(len);
  const int y = b - (1 << l) + 1;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    lo[k] = fminf(tab[refit_at(l, k, a)], tab[refit_at(l, k, y)]);
    hi[k] = fmaxf(tab[refit_at(l, D + k, a)], tab[refit_at(l, D + k, y)]);
  }
#pragma unroll
  for (int k = D; k < 3; ++k) { lo[k] = 0.f; hi[k] = 0.f; }
}

template <class Node>
__device__ __forceinline__ void refit_escape(Node* nodes, int link, const float* lo, const float* hi,
                                             unsigned* __restrict__ arrivals, int* __restrict__ up_list,
                                             unsigned* __restrict__ up_count) {
  const int node = link >> 1;
  put_child_box(nodes, node, link & 1, lo, hi);
  // relaxed: nothing in this launch reads the boxes; k_refit_up (the next
  // launch) sees them all
  if (atomicAdd(&arrivals[node], 1u) != 0) up_list[atomicAdd(up_count, 1u)] = node;
}

template <class Node, int D>
__global__ void __launch_bounds__(kRefitThreads)
k_refit(const float4* __restrict__ spts, long long n, Node* nodes, const int2* __restrict__ range,
        const int* __restrict__ node_parent, const int* __restrict__ leaf_parent, unsigned* __restrict__ arrivals,
        Box3* __restrict__ root_box, int* __restrict__ up_list, unsigned* __restrict__ up_count) {
  extern __shared__ __align__(16) float tab[];   // [level][slot][lo D, hi D]
  __shared__ int2 s_range[kRefitThreads];
  const int t = threadIdx.x;
  const long long B = (long long)blockIdx.x * kRefitThreads;
  const int cnt = (int)min((long long)kRefitThreads, n - B);
  const long long i = B + t;   // this thread's slot and internal node
  float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
  if (t < cnt) {
    p = spts[i];
    tab[refit_at(0, 0, t)] = p.x; tab[refit_at(0, 1, t)] = p.y;
    tab[refit_at(0, D, t)] = p.x; tab[refit_at(0, D + 1, t)] = p.y;
    if (D == 3) { tab[refit_at(0, 2, t)] = p.z; tab[refit_at(0, 5, t)] = p.z; }
  }
  s_range[t] = i < n - 1 ? range[i] : make_int2(-1, -1);
  __syncthreads();
  for (int l = 1; l < kRefitLevels && (1 << l) <= cnt; ++l) {
    const int h = 1 << (l - 1);
    if (t + (1 << l) <= cnt) {
#pragma unroll
      for (int k = 0; k < D; ++k) {
        tab[refit_at(l, k, t)] = fminf(tab[refit_at(l - 1, k, t)], tab[refit_at(l - 1, k, t + h)]);
        tab[refit_at(l, D + k, t)] = fmaxf(tab[refit_at(l - 1, D + k, t)], tab[refit_at(l - 1, D + k, t + h)]);
      }
    }
    __syncthreads();
  }
  const long long E = B + cnt;
  auto inside = [&](int node) -> bool {
    if (node < B || node >= E) return false;
    const int2 r = s_range[node - B];
    return r.x >= B && r.y < E;
  };
  if (i < n - 1) {
    const int2 r = s_range[t];
    if (r.x >= B && r.y < E) {
      const int lref = nodes[i].ref.x;
      const int gamma = lref >= 0 ? lref : ~lref;
      float alo[3], ahi[3], blo[3], bhi[3];
      refit_query<D>(tab, r.x - (int)B, gamma - (int)B, alo, ahi);
      refit_query<D>(tab, gamma + 1 - (int)B, r.y - (int)B, blo, bhi);
      put_node_boxes(nodes, (int)i, alo, ahi, blo, bhi);
#pragma unroll
      for (int k = 0; k < 3; ++k) { alo[k] = fminf(alo[k], blo[k]); ahi[k] = fmaxf(ahi[k], bhi[k]); }
      if (i == 0) {
        for (int k = 0; k < 3; ++k) { root_box->lo[k] = alo[k]; root_box->hi[k] = ahi[k]; }
      } else {
        const int link = node_parent[i];
        if (!inside(link >> 1)) refit_escape(nodes, link, alo, ahi, arrivals, up_list, up_count);
      }
    }
  }
  if (t < cnt) {
    const int link = leaf_parent[i];
    if (!inside(link >> 1)) {
      const float lo[3] = {p.x, p.y, D == 3 ? p.z : 0.f};
      refit_escape(nodes, link, lo, lo, arrivals, up_list, up_count);
    }
  }
}

// The upper tree: one thread per node listed by k_refit (both children done),
// climbing with the acq_rel arrival protocol until it arrives first.
template <class Node>
__global__ void __launch_bounds__(256)
k_refit_up(Node* nodes, const int* __restrict__ node_parent, unsigned* __restrict__ arrivals,
           const int* __restrict__ up_list, const unsigned* __restrict__ up_count, Box3* __restrict__ root_box) {
  const unsigned cnt = *up_count;
  for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += gridDim.x * blockDim.x) {
    int node = up_list[t];
    float lo[3], hi[3];
    for (;;) {
      get_union_box(nodes, node, lo, hi);
      if (node == 0) {
        for (int k = 0; k < 3; ++k) { root_box->lo[k] = lo[k]; root_box->hi[k] = hi[k]; }
        break;
      }
      const int link = node_parent[node];
      node = link >> 1;
      put_child_box(nodes, node, link & 1, lo, hi);
      // acq_rel: the first arrival's box is released by its increment and the
      // second arrival acquires it with its own (no full fences needed)
      unsigned prev;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(&arrivals[node]) : "memory");
      if (prev == 0) break;   // first arrival: sibling not done yet
    }
  }
}

// Node heights (leaf 0, internal 1 + the higher child) by the same arrival climb
// as the refit: the second thread to reach a node knows both subtrees are done.
// Feeds the export of the reference's level schedule (bvh.py:204-238, 293-302);
// the solve itself never needs it.
__global__ void k_node_heights(const int* __restrict__ leaf_parent, const int* __restrict__ node_parent, long long n,
                               unsigned* __restrict__ arrivals, unsigned* __restrict__ height) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= n || n < 2) return;
  unsigned h = 0;
  int link = leaf_parent[s];
  for (;;) {
    const int node = link >> 1;
    atomicMax(&height[node], h + 1);
    unsigned prev;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(&arrivals[node]) : "memory");
    if (prev == 0 || node == 0) return;
    h = atomicOr(&height[node], 0u);
    link = node_parent[node];
  }
}

__global__ void k_u32_to_u64(const unsigned* __restrict__ a, long long n, unsigned long long* __restrict__ out) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[i];
}

__global__ void k_u32_to_i64(const unsigned* __restrict__ a, long long n, long long* __restrict__ out) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[i];
}

// starts[k] = first position of height k + 1 in the ascending heights (np.searchsorted, left), and
// starts[hmax] = m (bvh.py:293-302).  Heights start at 1, so starts[0] = 0.
__global__ void k_level_starts(const unsigned long long* __restrict__ hs, const unsigned* __restrict__ order, long long m,
                               long long* __restrict__ starts, long long* __restrict__ order_out) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= m) return;
  order_out[i] = order[i];
  const unsigned long long h = hs[i], hp = i > 0 ? hs[i - 1] : 0;
  for (unsigned long long j = hp + 1; j <= h; ++j) starts[j - 1] = i;
  if (i == m - 1) starts[h] = m;
}

// Reference-layout export of the tree (bvh.py:39-75) for parity tests.
template <class Node>
__global__ void k_export_tree(const Node* __restrict__ nodes, const int* __restrict__ node_parent,
                              const int* __restrict__ leaf_parent, long long n, const Box3* __restrict__ root_box,
                              long long* left, long long* right, long long* parent, long long* lparent,
                              float* box_lo, float* box_hi, int d) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long m = n - 1;
  if (i < n) lparent[i] = m > 0 ? (long long)(leaf_parent[i] >> 1) : -1;
  if (i >= m) return;
  int4 r = nodes[i].ref;
  left[i] = r.x >= 0 ? (long long)r.x : m + (long long)(~r.x);
  right[i] = r.y >= 0 ? (long long)r.y : m + (long long)(~r.y);
  parent[i] = i == 0 ? -1 : (long long)(node_parent[i] >> 1);
  float lo[3], hi[3];
  if (i == 0) {
    for (int k = 0; k < 3; ++k) { lo[k] = root_box->lo[k]; hi[k] = root_box->hi[k]; }
  } else {
    int link = node_parent[i];
    int p = link >> 1, side = link & 1;
    const float* f = reinterpret_cast<const float*>(&nodes[p]);
    const float* o = f + side;   // interleaved children (common.cuh)
    if (sizeof(Node) == sizeof(Node3)) {
      lo[0] = o[0]; lo[1] = o[2]; lo[2] = o[4]; hi[0] = o[6]; hi[1] = o[8]; hi[2] = o[10];
    } else {
      lo[0] = o[0]; lo[1] = o[2]; hi[0] = o[4]; hi[1] = o[6]; lo[2] = hi[2] = 0.f;
    }
  }
  for (int k = 0; k < d; ++k) { box_lo[i * d + k] = lo[k]; box_hi[i * d + k] = hi[k]; }
}

}  // namespace emst
