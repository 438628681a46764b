// radix_sort.cuh -- stable onesweep LSD radix sort of u64 keys with u32 values.
//
// Same result as np.argsort(keys, kind="stable") when the values start as the
// identity (bvh.py:317): equal keys keep their input order.
//
//   1. k_digit_histograms: one read of the keys builds all eight 8-bit digit
//      histograms at once (shared-memory atomics, then one global add per bin).
//   2. k_digit_offsets: exclusive scan per digit; a pass whose digit is the same
//      for every key is skipped (its counting sort would be the identity).
//   3. k_onesweep: per active digit, one kernel reads 4096 keys per tile, ranks
//      them stably inside the tile (warp match_any + per-warp digit counters),
//      resolves the tile's global digit offsets with decoupled look-back over
//      the previous tiles, stages the tile in shared memory in sorted order and
//      writes it out digit-run-contiguous (coalesced).
#pragma once
#include "common.cuh"

namespace emst {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortItems = 16;
constexpr int kSortTile = kSortThreads * kSortItems;   // 4096 keys
constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;
constexpr int kMaxPasses = 8;

constexpr unsigned kSortFlagAgg = 1u << 30;
constexpr unsigned kSortFlagPrefix = 2u << 30;
constexpr unsigned kSortValueMask = (1u << 30) - 1;

__global__ void __launch_bounds__(kSortThreads)
k_digit_histograms(const unsigned long long* __restrict__ keys, long long n, int passes, unsigned* __restrict__ hist) {
  __shared__ unsigned s_hist[kMaxPasses][kRadix];
  for (int i = threadIdx.x; i < kMaxPasses * kRadix; i += blockDim.x) (&s_hist[0][0])[i] = 0;
  __syncthreads();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned long long k = keys[i];
    for (int p = 0; p < passes; ++p) atomicAdd(&s_hist[p][(k >> (p * kRadixBits)) & (kRadix - 1)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kRadix; i += blockDim.x) {
    unsigned c = (&s_hist[0][0])[i];
    if (c) atomicAdd(&hist[i], c);
  }
}

// One block of kRadix threads per pass: exclusive offsets + "pass is identity" bit.
__global__ void k_digit_offsets(const unsigned* __restrict__ hist, long long n, unsigned* __restrict__ offsets,
                                unsigned* __restrict__ active_mask) {
  __shared__ unsigned s[kRadix];
  __shared__ int s_trivial;
  const int p = blockIdx.x, t = threadIdx.x;
  unsigned c = hist[p * kRadix + t];
  if (t == 0) s_trivial = 0;
  s[t] = c;
  __syncthreads();
  if ((long long)c == n) s_trivial = 1;
  for (int o = 1; o < kRadix; o <<= 1) {
    unsigned v = t >= o ? s[t - o] : 0u;
    __syncthreads();
    s[t] += v;
    __syncthreads();
  }
  offsets[p * kRadix + t] = s[t] - c;
  if (t == 0 && !s_trivial) atomicOr(active_mask, 1u << p);
}

struct SortSmem {
  unsigned long long keys[kSortTile];
  unsigned vals[kSortTile];
  unsigned whist[kSortWarps][kRadix];
  unsigned tile_excl[kRadix];
  unsigned long long global_base[kRadix];
  unsigned scan_tmp[kRadix];
  long long tile;
};

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <bool kIotaValues>
__global__ void __launch_bounds__(kSortThreads)
k_onesweep(const unsigned long long* __restrict__ keys_in, const unsigned* __restrict__ vals_in,
           unsigned long long* __restrict__ keys_out, unsigned* __restrict__ vals_out, long long n, int shift,
           const unsigned* __restrict__ digit_offset, unsigned* __restrict__ status, unsigned* __restrict__ ticket) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SortSmem& sm = *reinterpret_cast<SortSmem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) sm.tile = (long long)atomicAdd(ticket, 1u);
  for (int i = tid; i < kSortWarps * kRadix; i += kSortThreads) (&sm.whist[0][0])[i] = 0;
  __syncthreads();
  const long long tile = sm.tile;
  const long long base = tile * kSortTile;
  const long long warp_base = base + warp * (32 * kSortItems);

  unsigned long long key[kSortItems];
  unsigned val[kSortItems];
  unsigned rank[kSortItems];
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    long long i = warp_base + j * 32 + lane;
    bool ok = i < n;
    key[j] = ok ? keys_in[i] : ~0ull;
    if (kIotaValues) val[j] = (unsigned)i;
    else val[j] = ok ? vals_in[i] : 0u;
  }
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    long long i = warp_base + j * 32 + lane;
    bool ok = i < n;
    unsigned d = ok ? (unsigned)((key[j] >> shift) & (kRadix - 1)) : (unsigned)kRadix;
    unsigned peers = __match_any_sync(0xffffffffu, d);
    unsigned before = 0;
    if (ok) before = sm.whist[warp][d];
    rank[j] = before + __popc(peers & lt);
    __syncwarp();
    if (ok && (peers & lt) == 0) sm.whist[warp][d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();

  // per digit (one thread each): prefix over warps, tile total, look-back
  {
    const int d = tid;
    unsigned run = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
      unsigned c = sm.whist[w][d];
      sm.whist[w][d] = run;
      run += c;
    }
    const unsigned total = run;
    unsigned* my = status + tile * kRadix + d;
    if (tile == 0) {
      atomicExch(my, kSortFlagPrefix | total);
      sm.global_base[d] = digit_offset[d];
    } else {
      atomicExch(my, kSortFlagAgg | total);
      unsigned excl = 0;
      long long t = tile - 1;
      for (;;) {
        unsigned s = *reinterpret_cast<volatile unsigned*>(status + t * kRadix + d);
        if ((s >> 30) == 0) continue;
        excl += s & kSortValueMask;
        if ((s >> 30) == 2) break;
        --t;
      }
      atomicExch(my, kSortFlagPrefix | (excl + total));
      sm.global_base[d] = (unsigned long long)digit_offset[d] + excl;
    }
    // tile-local exclusive digit starts (block scan over 256 digit totals)
    sm.scan_tmp[d] = total;
  }
  __syncthreads();
  for (int o = 1; o < kRadix; o <<= 1) {
    unsigned v = tid >= o ? sm.scan_tmp[tid - o] : 0u;
    __syncthreads();
    sm.scan_tmp[tid] += v;
    __syncthreads();
  }
  {
    unsigned incl = sm.scan_tmp[tid];
    unsigned tot = incl - (tid > 0 ? sm.scan_tmp[tid - 1] : 0u);
    __syncthreads();
    sm.tile_excl[tid] = incl - tot;
  }
  __syncthreads();

  // stage in tile-sorted order
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    long long i = warp_base + j * 32 + lane;
    if (i < n) {
      unsigned d = (unsigned)((key[j] >> shift) & (kRadix - 1));
      unsigned pos = sm.tile_excl[d] + sm.whist[warp][d] + rank[j];
      sm.keys[pos] = key[j];
      sm.vals[pos] = val[j];
    }
  }
  __syncthreads();
  const long long remain = n - base;
  const int count = remain < kSortTile ? (int)remain : kSortTile;
  for (int i = tid; i < count; i += kSortThreads) {
    unsigned long long k = sm.keys[i];
    unsigned d = (unsigned)((k >> shift) & (kRadix - 1));
    unsigned long long dst = sm.global_base[d] + (unsigned)(i - sm.tile_excl[d]);
    keys_out[dst] = k;
    vals_out[dst] = sm.vals[i];
  }
}

inline long long sort_tiles(long long n) { return (n + kSortTile - 1) / kSortTile; }

}  // namespace emst
