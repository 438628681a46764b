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

#ifndef EMST_SORT_THREADS
#define EMST_SORT_THREADS 256
#endif
#ifndef EMST_SORT_ITEMS
#define EMST_SORT_ITEMS 16
#endif
constexpr int kSortThreads = EMST_SORT_THREADS;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortItems = EMST_SORT_ITEMS;
constexpr int kSortTile = kSortThreads * kSortItems;   // 4096 keys
constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;
constexpr int kMaxPasses = 8;

constexpr unsigned kSortFlagAgg = 1u << 30;
constexpr unsigned kSortFlagPrefix = 2u << 30;
constexpr unsigned kSortValueMask = (1u << 30) - 1;

template <class K>
__global__ void __launch_bounds__(kSortThreads)
k_digit_histograms(const K* __restrict__ keys, long long n, int passes, unsigned* __restrict__ hist) {
  __shared__ unsigned s_hist[kMaxPasses][kRadix];
  for (int i = threadIdx.x; i < kMaxPasses * kRadix; i += blockDim.x) (&s_hist[0][0])[i] = 0;
  __syncthreads();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[i];
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

template <class K>
struct SortSmemT {
  K keys[kSortTile];
  unsigned vals[kSortTile];
  unsigned short whist[kSortWarps][kRadix];   // per-warp digit counts, then exclusive warp offsets
  unsigned tile_excl[kRadix];
  unsigned long long global_base[kRadix];
  long long tile;
};
using SortSmem = SortSmemT<unsigned long long>;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ unsigned warp_incl_sum_u32(unsigned v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned t = __shfl_up_sync(0xffffffffu, v, o);
    if ((int)(threadIdx.x & 31) >= o) v += t;
  }
  return v;
}

#ifndef EMST_SORT_MINB
#define EMST_SORT_MINB 4
#endif

// What a pass writes besides the values: the keys as they are, only their high
// 32 bits (the passes left read nothing below them), or nothing (last pass).
enum SortOut { kOutSame = 0, kOutHigh32 = 1, kOutNone = 2 };
template <class K, int O> struct SortOutKey { using type = K; };
template <class K> struct SortOutKey<K, kOutHigh32> { using type = unsigned; };
template <class K> struct SortOutKey<K, kOutNone> { using type = unsigned; };

// One counting-sort pass over `shift`'s 8-bit digit of K keys.  Per tile of kSortTile keys:
//   1. warp-private stable ranks: the lanes holding the same digit are found
//      with 8 ballots (one per digit bit); the lowest bumps the warp's counter
//      in shared memory by the group size and broadcasts the old value (items
//      are visited in input order, so equal digits keep their input order);
//   2. per digit: prefix over the warps and the tile total, which is published
//      at once for the tiles behind;
//   3. keys and values are staged in shared memory in tile-sorted order (values
//      are only read here, so the ranking holds just the keys and packed ranks)
//      -- this is the work that overlaps the predecessors' progress --
//   4. decoupled look-back for each digit's global start, then the tile is
//      written out digit-run-contiguous (keys converted as SortOut says).
template <class K, int kOut, bool kIotaValues>
__global__ void __launch_bounds__(kSortThreads, EMST_SORT_MINB)
k_onesweep(const K* __restrict__ keys_in, const unsigned* __restrict__ vals_in,
           typename SortOutKey<K, kOut>::type* __restrict__ keys_out, unsigned* __restrict__ vals_out, long long n,
           int shift, const unsigned* __restrict__ digit_offset, unsigned* __restrict__ status,
           unsigned* __restrict__ ticket) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SortSmemT<K>& sm = *reinterpret_cast<SortSmemT<K>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // peer-mask bins of the ranking, two sets per warp (alternating items), in the
  // key staging area, which is only written after the ranking
  static_assert(sizeof(SortSmemT<K>::keys) >= 2 * kSortWarps * kRadix * sizeof(unsigned), "match bins");
  unsigned* const mbin = reinterpret_cast<unsigned*>(sm.keys);
  if (tid == 0) sm.tile = (long long)atomicAdd(ticket, 1u);
  for (int i = tid; i < kSortWarps * kRadix / 2; i += kSortThreads) reinterpret_cast<unsigned*>(&sm.whist[0][0])[i] = 0u;
  for (int i = tid; i < 2 * kSortWarps * kRadix; i += kSortThreads) mbin[i] = 0u;
  __syncthreads();
  const long long tile = sm.tile;
  const long long base = tile * kSortTile;
  const long long warp_base = base + warp * (32 * kSortItems);

  K key[kSortItems];
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const long long i = warp_base + j * 32 + lane;
    key[j] = i < n ? keys_in[i] : (K)~(K)0;
  }
  const unsigned lt = lanemask_lt();
  unsigned rank2[kSortItems / 2];   // two 16-bit ranks per register
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    // Stable warp-local rank: every lane ORs its bit into its digit's peer mask,
    // the lowest lane of each digit group bumps the warp's counter by the group
    // size, and a lane's rank is the counter's old value plus its lower peers
    // (items are visited in input order, so equal digits keep their order).
    // The mask is cleared by its leader; the next item uses the other bin set,
    // so the clear never races with the next ORs.
    const long long i = warp_base + j * 32 + lane;
    const bool ok = i < n;
    const unsigned d = (unsigned)((key[j] >> shift) & (kRadix - 1));
    unsigned* bin = mbin + ((j & 1) * kSortWarps + warp) * kRadix + d;
    if (ok) atomicOr(bin, 1u << lane);
    __syncwarp();
    const unsigned peers = ok ? *reinterpret_cast<volatile unsigned*>(bin) : 0u;
    const int leader = __ffs(peers) - 1;   // (an invalid lane has peers = 0: leader -1)
    unsigned before = 0;
    if (ok && lane == leader) {
      before = sm.whist[warp][d];
      sm.whist[warp][d] = (unsigned short)(before + __popc(peers));
    }
    __syncwarp();   // (every lane has read its mask and the counters are updated)
    if (ok && lane == leader) *bin = 0u;
    before = __shfl_sync(0xffffffffu, before, leader < 0 ? 0 : leader);
    const unsigned r = before + __popc(peers & lt);
    if (j & 1) rank2[j >> 1] |= r << 16; else rank2[j >> 1] = r;
  }
  __syncthreads();

  // per digit (one thread each): prefix over warps, tile total published
  const int dg = tid;
  unsigned total;
  {
    unsigned run = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
      const unsigned c = sm.whist[w][dg];
      sm.whist[w][dg] = (unsigned short)run;
      run += c;
    }
    total = run;
    atomicExch(status + tile * kRadix + dg, (tile == 0 ? kSortFlagPrefix : kSortFlagAgg) | total);
    // tile-local exclusive digit starts: block scan of the 256 digit totals
    const unsigned incl = warp_incl_sum_u32(total);
    if (lane == 31) sm.tile_excl[warp] = incl;   // (scratch: per-warp sums)
    __syncthreads();
    if (warp == 0) {
      const unsigned ws = lane < kSortWarps ? sm.tile_excl[lane] : 0u;
      const unsigned wi = warp_incl_sum_u32(ws);
      if (lane < kSortWarps) sm.tile_excl[lane] = wi - ws;
    }
    __syncthreads();
    const unsigned woff = sm.tile_excl[warp];
    __syncthreads();
    sm.tile_excl[dg] = woff + incl - total;
  }
  __syncthreads();

  // stage keys and values in tile-sorted order
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const long long i = warp_base + j * 32 + lane;
    if (i < n) {
      const unsigned d = (unsigned)((key[j] >> shift) & (kRadix - 1));
      const unsigned r = (rank2[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
      const unsigned pos = sm.tile_excl[d] + sm.whist[warp][d] + r;
      sm.keys[pos] = key[j];
      sm.vals[pos] = kIotaValues ? (unsigned)i : vals_in[i];
    }
  }

  // look-back: global start of this tile's run of each digit
  if (tile == 0) {
    sm.global_base[dg] = digit_offset[dg];
  } else {
    unsigned excl = 0;
    long long t = tile - 1;
    for (;;) {
      const unsigned s = *reinterpret_cast<volatile unsigned*>(status + t * kRadix + dg);
      if ((s >> 30) == 0) continue;
      excl += s & kSortValueMask;
      if ((s >> 30) == 2) break;
      --t;
    }
    atomicExch(status + tile * kRadix + dg, kSortFlagPrefix | (excl + total));
    sm.global_base[dg] = (unsigned long long)digit_offset[dg] + excl;
  }
  __syncthreads();
  const long long remain = n - base;
  const int count = remain < kSortTile ? (int)remain : kSortTile;
  for (int i = tid; i < count; i += kSortThreads) {
    const K k = sm.keys[i];
    const unsigned d = (unsigned)((k >> shift) & (kRadix - 1));
    const unsigned long long dst = sm.global_base[d] + (unsigned)(i - sm.tile_excl[d]);
    if (kOut == kOutSame) keys_out[dst] = (typename SortOutKey<K, kOut>::type)k;
    else if (kOut == kOutHigh32) keys_out[dst] = (unsigned)((unsigned long long)k >> 32);
    vals_out[dst] = sm.vals[i];
  }
}

inline long long sort_tiles(long long n) { return (n + kSortTile - 1) / kSortTile; }

}  // namespace emst
