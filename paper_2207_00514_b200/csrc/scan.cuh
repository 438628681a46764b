// scan.cuh -- single-pass exclusive prefix scan with decoupled look-back.
//
// One launch scans n items: tiles take a ticket from an atomic counter (so every
// tile that waits has only resident predecessors), publish their aggregate,
// and one warp looks back 32 predecessors at a time.  Payloads are u64 with a
// 62-bit value; the top two bits of each tile status word are the flag.
// Loader(i) -> u64 and Storer(i, exclusive, value) are fused by the caller, so
// the scan costs one read and one write of the scanned stream.
#pragma once
#include "common.cuh"

namespace emst {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagPrefix = 2ull << 62;
constexpr unsigned long long kValueMask = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}
__device__ __forceinline__ void st_volatile_u64(unsigned long long* p, unsigned long long v) {
  *reinterpret_cast<volatile unsigned long long*>(p) = v;
}

__device__ __forceinline__ unsigned long long warp_incl_sum(unsigned long long v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned long long t = __shfl_up_sync(0xffffffffu, v, o);
    if ((int)lane_id() >= o) v += t;
  }
  return v;
}

// Scratch per scan launch: status[num_tiles] and a ticket counter, zeroed
// before launch (cudaMemsetAsync of (num_tiles + 1) u64).
template <class Loader, class Storer>
__global__ void __launch_bounds__(kScanThreads)
k_scan(long long n, unsigned long long* status, unsigned long long* ticket, Loader load, Storer store,
       unsigned long long* total_out) {
  __shared__ unsigned long long s_val[kScanTile];
  __shared__ unsigned long long s_warp[kScanThreads / 32];
  __shared__ unsigned long long s_prefix;
  __shared__ long long s_tile;
  const int tid = threadIdx.x;
  if (tid == 0) s_tile = (long long)atomicAdd(ticket, 1ull);
  __syncthreads();
  const long long tile = s_tile;
  const long long base = tile * kScanTile;

  // striped loads (coalesced), blocked per-thread reduction through smem
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    long long i = base + j * kScanThreads + tid;
    s_val[j * kScanThreads + tid] = i < n ? load(i) : 0ull;
  }
  __syncthreads();
  unsigned long long mine[kScanItems];
  unsigned long long tsum = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    mine[j] = s_val[tid * kScanItems + j];
    tsum += mine[j];
  }
  unsigned long long incl = warp_incl_sum(tsum);
  if (lane_id() == 31) s_warp[tid >> 5] = incl;
  __syncthreads();
  if (tid < 32) {
    unsigned long long w = tid < kScanThreads / 32 ? s_warp[tid] : 0ull;
    unsigned long long wi = warp_incl_sum(w);
    if (tid < kScanThreads / 32) s_warp[tid] = wi - w;   // exclusive warp offsets
    unsigned long long agg = __shfl_sync(0xffffffffu, wi, kScanThreads / 32 - 1);
    // publish, then look back
    if (tile == 0) {
      if (tid == 0) { st_volatile_u64(&status[0], kFlagPrefix | (agg & kValueMask)); s_prefix = 0; }
    } else {
      if (tid == 0) st_volatile_u64(&status[tile], kFlagAgg | (agg & kValueMask));
      unsigned long long excl = 0;
      long long t = tile - 1;
      for (;;) {
        long long idx = t - (long long)tid;
        unsigned long long st = idx >= 0 ? ld_volatile_u64(&status[idx]) : kFlagPrefix;
        while (__any_sync(0xffffffffu, (st >> 62) == 0)) {
          if ((st >> 62) == 0) st = ld_volatile_u64(&status[idx]);
        }
        unsigned pm = __ballot_sync(0xffffffffu, (st >> 62) == 2);
        int stop = pm ? __ffs(pm) - 1 : 31;
        unsigned long long c = (int)tid <= stop ? (st & kValueMask) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        excl += c;
        if (pm) break;
        t -= 32;
      }
      if (tid == 0) { st_volatile_u64(&status[tile], kFlagPrefix | ((excl + agg) & kValueMask)); s_prefix = excl; }
    }
    if (total_out && tid == 0 && base + kScanTile >= n) {
      // the last tile knows the grand total once its prefix is resolved
      *total_out = (tile == 0 ? 0ull : s_prefix) + agg;
    }
  }
  __syncthreads();
  unsigned long long run = s_prefix + s_warp[tid >> 5] + (incl - tsum);
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    s_val[tid * kScanItems + j] = run;
    run += mine[j];
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    long long i = base + j * kScanThreads + tid;
    if (i < n) store(i, s_val[j * kScanThreads + tid]);
  }
}

inline long long scan_tiles(long long n) { return (n + kScanTile - 1) / kScanTile; }

}  // namespace emst
