// scan.cuh -- single-pass exclusive prefix scan with decoupled look-back.
//
// One launch scans n items.  Tiles take a ticket from an atomic counter (so a
// tile that waits only waits on resident predecessors), publish their
// aggregate, and one warp looks back 32 predecessors at a time.
//
// Items are BLOCKED: thread t of a tile owns kScanItems consecutive items, so
// an operation can fetch them with vector loads and issue all of its (often
// data-dependent) memory traffic for the 8 items at once instead of one
// latency chain per item.  The operation supplies
//   Op::T                      the value type (u32, or u64 with 62 value bits)
//   op.load(i0, cnt, v)        fill v[0..cnt) for items i0.. (side work allowed;
//                              called by every thread, cnt may be 0)
//   op.side(i0, cnt, v)        optional work that does not feed the scan, run
//                              after the tile's prefix is published (so the
//                              look-back chain of the tiles behind never waits
//                              on it); called by every thread
//   op.store(i0, cnt, v, ex)   ex = exclusive prefix of item i0 (threads with cnt 0
//                              call it too when Op::kWarpStore)
// Value arithmetic wraps (mod 2^32 for u32, mod 2^62 for u64), which is exact
// whenever every true prefix fits, so signed contributions are allowed.
#pragma once
#include "common.cuh"

namespace emst {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;
constexpr int kLookPerLane = 4;   // look-back window = 32 * 4 predecessor tiles

constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagPrefix = 2ull << 62;
constexpr unsigned long long kValueMask = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}
__device__ __forceinline__ void st_volatile_u64(unsigned long long* p, unsigned long long v) {
  *reinterpret_cast<volatile unsigned long long*>(p) = v;
}

template <class T>
__device__ __forceinline__ T warp_incl_sum(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T t = __shfl_up_sync(0xffffffffu, v, o);
    if ((int)lane_id() >= o) v += t;
  }
  return v;
}

template <class T> __device__ __forceinline__ unsigned long long pack_status(unsigned long long flag, T v) {
  return flag | ((unsigned long long)v & kValueMask);
}
template <class T> __device__ __forceinline__ T unpack_status(unsigned long long s) { return (T)(s & kValueMask); }

// Exclusive prefix (global) of this thread's `mine` within the scan; `tile` is
// the ticket.  All threads of the block must call it.  *tile_total receives the
// inclusive prefix at the end of the tile.
template <class T>
__device__ __forceinline__ T tile_exclusive(T mine, long long tile, unsigned long long* status, T* tile_total) {
  __shared__ T s_warp[kScanThreads / 32];
  __shared__ T s_prefix;
  __shared__ T s_total;
  const int tid = threadIdx.x;
  const T incl = warp_incl_sum(mine);
  if (lane_id() == 31) s_warp[tid >> 5] = incl;
  __syncthreads();
  if (tid < 32) {
    const T w = tid < kScanThreads / 32 ? s_warp[tid] : T(0);
    const T wi = warp_incl_sum(w);
    if (tid < kScanThreads / 32) s_warp[tid] = wi - w;   // exclusive warp offsets
    const T agg = __shfl_sync(0xffffffffu, wi, kScanThreads / 32 - 1);
    if (tile == 0) {
      if (tid == 0) {
        st_volatile_u64(&status[0], pack_status<T>(kFlagPrefix, agg));
        s_prefix = T(0);
        s_total = agg;
      }
    } else {
      if (tid == 0) st_volatile_u64(&status[tile], pack_status<T>(kFlagAgg, agg));
      // Look back kLookback tiles per step (lane l reads tiles t-1-4l .. t-4-4l),
      // so the prefix front advances 128 tiles per round trip instead of 32.
      T excl = T(0);
      long long t = tile - 1;
      for (;;) {
        unsigned long long st[kLookPerLane];
#pragma unroll
        for (int k = 0; k < kLookPerLane; ++k) {
          const long long idx = t - (long long)tid * kLookPerLane - k;
          st[k] = idx >= 0 ? ld_volatile_u64(&status[idx]) : kFlagPrefix;
        }
        for (;;) {
          bool waiting = false;
#pragma unroll
          for (int k = 0; k < kLookPerLane; ++k) waiting |= (st[k] >> 62) == 0;
          if (!__any_sync(0xffffffffu, waiting)) break;
#pragma unroll
          for (int k = 0; k < kLookPerLane; ++k) {
            const long long idx = t - (long long)tid * kLookPerLane - k;
            if ((st[k] >> 62) == 0) st[k] = ld_volatile_u64(&status[idx]);
          }
        }
        // this lane's sum back to (and including) its nearest inclusive prefix
        T c = T(0);
        bool has_prefix = false;
#pragma unroll
        for (int k = 0; k < kLookPerLane; ++k) {
          if (!has_prefix) {
            c += unpack_status<T>(st[k]);
            has_prefix = (st[k] >> 62) == 2;
          }
        }
        const unsigned pm = __ballot_sync(0xffffffffu, has_prefix);
        const int stop = pm ? __ffs(pm) - 1 : 31;
        if ((int)tid > stop) c = T(0);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        excl += c;
        if (pm) break;
        t -= 32 * kLookPerLane;
      }
      if (tid == 0) {
        st_volatile_u64(&status[tile], pack_status<T>(kFlagPrefix, excl + agg));
        s_prefix = excl;
        s_total = excl + agg;
      }
    }
  }
  __syncthreads();
  *tile_total = s_total;
  return s_prefix + s_warp[tid >> 5] + (incl - mine);
}

// Block-wide exclusive scan of one value per thread (no look-back); returns the
// thread's exclusive offset and the block total in *total.
template <class T>
__device__ __forceinline__ T block_exclusive(T mine, T* total) {
  __shared__ T s_w[kScanThreads / 32];
  __shared__ T s_tot;
  const int tid = threadIdx.x;
  const T incl = warp_incl_sum(mine);
  __syncthreads();   // s_w may still be read from the previous call
  if (lane_id() == 31) s_w[tid >> 5] = incl;
  __syncthreads();
  if (tid < 32) {
    const T w = tid < kScanThreads / 32 ? s_w[tid] : T(0);
    const T wi = warp_incl_sum(w);
    if (tid < kScanThreads / 32) s_w[tid] = wi - w;
    if (tid == kScanThreads / 32 - 1) s_tot = wi;
  }
  __syncthreads();
  *total = s_tot;
  return s_w[tid >> 5] + (incl - mine);
}

// Persistent segmented scan: block b owns the contiguous segment
// [b * seg, (b + 1) * seg) (seg a multiple of kScanTile) and walks it twice --
// once to reduce it, once to scan it -- with a single decoupled look-back among
// the blocks in between (every block is resident, the grid is sized by the
// occupancy).  The input is read twice, but there is no per-tile serial
// look-back chain.  status[gridDim.x] must be zeroed before the launch; the
// grand total goes to *total_out when it is given.
// 5 resident blocks per SM (<= 51 registers): the round scans at 37M blobs 3D 2.67 -> 2.57 ms
// summed (4 blocks: the compiler's own 63 registers; 6: 2.69; 8: 3.4)
#ifndef EMST_SCAN_MINB
#define EMST_SCAN_MINB 5
#endif
template <class Op>
__global__ void __launch_bounds__(kScanThreads, EMST_SCAN_MINB)
k_scan(long long n, long long seg, unsigned long long* status, Op op, unsigned long long* total_out) {
  using T = typename Op::T;
  const long long b = blockIdx.x;
  const long long s0 = b * seg;
  const long long s1 = min(n, s0 + seg);
  T acc = T(0);
  for (long long base = s0; base < s1; base += kScanTile) {
    const long long i0 = base + (long long)threadIdx.x * kScanItems;
    const int cnt = i0 >= s1 ? 0 : (s1 - i0 < kScanItems ? (int)(s1 - i0) : kScanItems);
    T v[kScanItems];
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) v[j] = T(0);
    op.load(i0, cnt, v);
    if constexpr (Op::kCached) { if (cnt > 0) op.put(i0, cnt, v); }
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) acc += v[j];
  }
  T seg_total;
  const T my_ex = tile_exclusive<T>(acc, b, status, &seg_total);   // (only its segment prefix is used)
  __shared__ T s_base;
  if (threadIdx.x == 0) s_base = my_ex;   // thread 0: exclusive prefix of the whole segment
  __syncthreads();
  T run = s_base;
  for (long long base = s0; base < s1; base += kScanTile) {
    const long long i0 = base + (long long)threadIdx.x * kScanItems;
    const int cnt = i0 >= s1 ? 0 : (s1 - i0 < kScanItems ? (int)(s1 - i0) : kScanItems);
    T v[kScanItems];
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) v[j] = T(0);
    if constexpr (Op::kCached) { if (cnt > 0) op.get(i0, cnt, v); }
    else op.load(i0, cnt, v);
    T mine = T(0);
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) mine += v[j];
    T tile_total;
    const T off = block_exclusive<T>(mine, &tile_total);
    op.side(i0, cnt, v);
    if constexpr (Op::kWarpStore) op.store(i0, cnt, v, run + off);   // (every thread)
    else if (cnt > 0) op.store(i0, cnt, v, run + off);
    run += tile_total;
  }
  if (total_out && threadIdx.x == 0 && s1 >= n && s0 < n) *total_out = (unsigned long long)seg_total;
  if (total_out && threadIdx.x == 0 && n == 0 && b == 0) *total_out = 0ull;
}

inline long long scan_tiles(long long n) { return (n + kScanTile - 1) / kScanTile; }

// Blocked 8-item loads/stores of 32-bit values (i0 is a multiple of 8, so the
// full-count case is two aligned 16-byte accesses).
template <class V>
__device__ __forceinline__ void load8(const V* __restrict__ a, long long i0, int cnt, V* out) {
  static_assert(sizeof(V) == 4, "32-bit items");
  if (cnt == kScanItems) {
    const int4 x = __ldg(reinterpret_cast<const int4*>(a + i0));
    const int4 y = __ldg(reinterpret_cast<const int4*>(a + i0) + 1);
    const int r[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
#pragma unroll
    for (int j = 0; j < 8; ++j) out[j] = *reinterpret_cast<const V*>(&r[j]);
  } else {
#pragma unroll
    for (int j = 0; j < kScanItems; ++j)
      if (j < cnt) out[j] = a[i0 + j];
  }
}
template <class V>
__device__ __forceinline__ void store8(V* __restrict__ a, long long i0, int cnt, const V* in) {
  static_assert(sizeof(V) == 4, "32-bit items");
  if (cnt == kScanItems) {
    int r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = *reinterpret_cast<const int*>(&in[j]);
    reinterpret_cast<int4*>(a + i0)[0] = make_int4(r[0], r[1], r[2], r[3]);
    reinterpret_cast<int4*>(a + i0)[1] = make_int4(r[4], r[5], r[6], r[7]);
  } else {
#pragma unroll
    for (int j = 0; j < kScanItems; ++j)
      if (j < cnt) a[i0 + j] = in[j];
  }
}

}  // namespace emst
