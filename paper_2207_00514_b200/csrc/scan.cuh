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
//   op.store(i0, cnt, v, ex)   ex = exclusive prefix of item i0
// Value arithmetic wraps (mod 2^32 for u32, mod 2^62 for u64), which is exact
// whenever every true prefix fits, so signed contributions are allowed.
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
      T excl = T(0);
      long long t = tile - 1;
      for (;;) {
        const long long idx = t - (long long)tid;
        unsigned long long st = idx >= 0 ? ld_volatile_u64(&status[idx]) : kFlagPrefix;
        while (__any_sync(0xffffffffu, (st >> 62) == 0)) {
          if ((st >> 62) == 0) st = ld_volatile_u64(&status[idx]);
        }
        const unsigned pm = __ballot_sync(0xffffffffu, (st >> 62) == 2);
        const int stop = pm ? __ffs(pm) - 1 : 31;
        T c = (int)tid <= stop ? unpack_status<T>(st) : T(0);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        excl += c;
        if (pm) break;
        t -= 32;
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

// Scratch per scan launch: status[num_tiles] and a ticket counter, zeroed
// before launch (cudaMemsetAsync of (num_tiles + 1) u64).  The last tile
// writes the grand total to *total_out when it is given.
template <class Op>
__global__ void __launch_bounds__(kScanThreads)
k_scan(long long n, unsigned long long* status, unsigned long long* ticket, Op op, unsigned long long* total_out) {
  using T = typename Op::T;
  __shared__ long long s_tile;
  if (threadIdx.x == 0) s_tile = (long long)atomicAdd(ticket, 1ull);
  __syncthreads();
  const long long tile = s_tile;
  const long long i0 = tile * kScanTile + (long long)threadIdx.x * kScanItems;
  const int cnt = i0 >= n ? 0 : (n - i0 < kScanItems ? (int)(n - i0) : kScanItems);
  T v[kScanItems];
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) v[j] = T(0);
  op.load(i0, cnt, v);   // every thread calls it (cnt may be 0): ops may use warp collectives
  T mine = T(0);
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) mine += v[j];
  T total;
  const T ex = tile_exclusive<T>(mine, tile, status, &total);
  if (cnt > 0) op.store(i0, cnt, v, ex);
  if (total_out && threadIdx.x == 0 && (tile + 1) * kScanTile >= n) *total_out = (unsigned long long)total;
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
