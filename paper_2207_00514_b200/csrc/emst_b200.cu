// emst_b200.cu -- host orchestration and the C ABI (include/emst_b200.h).
//
// One context per (process, device) owns a stream, a capacity-sized device
// workspace (reused across calls) and, for world > 1, an NCCL communicator.
// The Boruvka loop keeps every array device-resident; the host reads back 24
// bytes per round (new component count, edge count, error bits) to steer it.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <functional>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/emst_b200.h"
#include "boruvka.cuh"
#include "core.cuh"
#include "build.cuh"
#include "radix_sort.cuh"
#include "hostio.h"
#include "textio.h"
#include "textparse.h"
#include "scan.cuh"

using namespace emst;

namespace {

struct Failure {
  int code;
  char msg[256];
};

[[noreturn]] void fail(int code, const char* fmt, ...) {
  Failure f;
  f.code = code;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(f.msg, sizeof(f.msg), fmt, ap);
  va_end(ap);
  throw f;
}

#define CK(x)                                                                                 \
  do {                                                                                        \
    cudaError_t e_ = (x);                                                                     \
    if (e_ != cudaSuccess) fail(EMST_ERR_CUDA, "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), \
                                __FILE__, __LINE__);                                          \
  } while (0)

#define NK(x)                                                                                   \
  do {                                                                                          \
    ncclResult_t r_ = (x);                                                                      \
    if (r_ != ncclSuccess) fail(EMST_ERR_NCCL, "%s: %s", #x, ncclGetErrorString(r_));           \
  } while (0)

template <class T>
struct HostBuf {   // page-locked host staging
  T* p = nullptr;
  size_t cap = 0;
  void ensure_host(size_t count) {
    if (count <= cap) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    CK(cudaMallocHost(&p, std::max<size_t>(count, 1) * sizeof(T)));
    cap = count;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
  }
};

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t cap = 0;
  void ensure(size_t count) {
    if (count <= cap) return;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    CK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
    cap = count;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

inline unsigned grid_for(long long n, int threads) { return (unsigned)std::max<long long>(1, (n + threads - 1) / threads); }

}  // namespace

#ifndef EMST_SEED1_W
#define EMST_SEED1_W 8   // round 1's Z-window of radius seeds
#endif
constexpr long long kIpermPart = 1ll << 23;   // inverse-permutation targets per scatter part (32 MB of iperm)
constexpr int kCounters = 16;   // [0] evals [1] scan total [2] err [3] overflow [4] work [5] visits
                                // [6] found [7] ties [8] frontier size [9] skipped queries [10] big tops [11] mid tie runs
                                // [12] slots of component 1 (last round) [13] the component left out
                                // [14] slots listed by the prefilter [15] refit nodes for the upper tree

struct emst_context {
  int device = 0, rank = 0, world = 1, vshards = 1;
  bool singleton_round = false;   // every component is one point (round 1 of a solve)
  int round = 0;                  // 1-based Boruvka round of the running solve (0 outside)
  int seed_window = 8;            // Z-order seed pairs (s +- 1..W) in solve rounds >= 2 (EMST_SEED_WINDOW)
  long long round_comps = 0;      // components entering the running round
  int seed_from = 2;
  int seed_window_2d = 4;         // the same in 2D (EMST_SEED_WINDOW_2D, <= 1: off)              // first round with window seeds (EMST_SEED_FROM)
  double skip_frac = 0.0;         // share of last round's queries settled before their first visit
  bool single_kernel = true;      // round 1 runs its own compiled traversal (EMST_SINGLE_KERNEL=0: the general one)
  double list_skip = 0.1;         // prefilter the queries when last round settled this share up front (EMST_LIST_SKIP)
  DevBuf<int> qlist;              // slots the prefilter kept
  int iperm_parts = 0;            // parts of the inverse-permutation scatter (0: by size, EMST_IPERM_PARTS)
  bool one_side = false;          // last round (2 components): run only the smaller component's queries
  bool last_round_one_side = true;   // EMST_ONE_SIDE=0 turns that off
  bool trace = false;             // per-round trace on stderr (EMST_TRACE=1; developer aid)
  int proof_from = 3;             // first round whose traversal records the full nearest-foreign proof (EMST_PROOF_FROM)
  ncclComm_t comm = nullptr;
  emst_exchange_fn exch_fn = nullptr;   // host exchange (world > 1 without NCCL)
  void* exch_user = nullptr;
  HostBuf<unsigned long long> exch_host;
  emst_host::Stager stager;          // pageable host <-> HBM pipeline of the host-pointer entry
  bool staging = true;               // EMST_STAGE=0: plain cudaMemcpyAsync of pageable memory (A/B)
  bool packed_out = true;            // EMST_PACKED=0: int64 rows straight from the device (A/B)
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  cudaStream_t copy_stream = nullptr;   // second copy engine: the weights D2H beside the edge chunks
  long long launches = 0;
  double traverse_ms = 0.0;
  long long traverse_launches = 0, traverse_queries = 0;
  int num_sms = 148;

  // build
  DevBuf<float> pts;
  DevBuf<Scene> scene;
  DevBuf<float> part_lo, part_hi;
  DevBuf<long long> part_bad;
  DevBuf<unsigned long long> k0, k1;
  DevBuf<unsigned> v0, v1;
  DevBuf<unsigned> sort_hist, sort_off, sort_status, sort_misc;
  DevBuf<float4> spts;
  DevBuf<unsigned> perm, iperm;
  DevBuf<unsigned char> nodes;   // Node2 / Node3 records
  DevBuf<int2> range;
  DevBuf<int> node_parent, leaf_parent, node_delta;
  DevBuf<int2> up;   // (parent link, prefix length) per internal node
  DevBuf<unsigned> arrivals;
  DevBuf<Box3> root_box;
  // rounds
  DevBuf<int> label, bprefix;
  DevBuf<float> nfn_lb;   // per slot: proven lower bound on the nearest-foreign distance
  DevBuf<int> top;
  DevBuf<int4> big_tops;           // top pure node per slot (T + 1, 0 = none); large ones to fill
  DevBuf<int> front[2];                // internal nodes still mixed after the last labelling
  // mutual reachability: core distance per slot; `core` points at it while a
  // mutual-reachability solve / building block runs, nullptr for Euclidean
  DevBuf<double> core_slot, core_tmp;
  const double* core = nullptr;
  long long front_n = -1;              // their count (-1: none yet, label every node)
  bool front_pending = false;
  int front_cur = 0;
  bool top_valid = false;              // top[] holds this round's values
  DevBuf<unsigned long long> ub;
  DevBuf<EdgeKey> best, shard_keys;
  DevBuf<int> succ, ptr, root, newid, fin;
  DevBuf<EdgeKey> eout;   // emitted edges: (u << 32 | v, weight bits)
  DevBuf<unsigned long long> xw, xuv;   // multi-GPU exchange
  DevBuf<unsigned long long> scan_scratch;
  DevBuf<long long> counters;   // [0] evals, [1] scan total, [2] err, [3] overflow
  DevBuf<long long> out_edges;
  DevBuf<double> out_w;
  DevBuf<double> pairwise;   // total-weight partial sums
  DevBuf<int2> tie_runs, tie_mid, tie_small;   // (start, length) of the 257..4096 / 9..32 / 33..256-edge equal-key runs
  long long* host_counters = nullptr;   // pinned mirror of `counters`
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  // deferred final emit (packed host output, EMST_EMIT_OVERLAP): the final order and its keys, and
  // one event per emitted chunk for the copies to wait on
  bool emit_overlap = true;
  bool emit_deferred = false;
  const unsigned* emit_order = nullptr;
  const unsigned* emit_key = nullptr;
  std::vector<cudaEvent_t> emit_ev;
  // Phase timers read back lazily: event pairs are recorded on the stream and
  // their times collected at the next stream sync the solve needs anyway (the
  // round's counter read), so timing adds no host round trip of its own.
  struct Timer {
    cudaEvent_t a, b;
    double* acc;      // += elapsed ms (or nullptr)
    bool trav;        // a traversal launch (traverse_ms, trace)
    int round;
    long long q0, q1;
  };
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_next = 0;
  std::vector<Timer> timers;
  size_t nodes_stride = 0;
  int dim = 0;
  long long n = 0;
  bool tree_valid = false;
  long long tree_token = 0;       // bumped by every build: names the tree the context holds
  cudaEvent_t merge_end = nullptr;  // the last merge's end (trace: device idle time to the next round)
  cudaEvent_t ev_counters = nullptr;   // the queued counter copy (read_counters_async)
  size_t counters_timers = 0;          // timers recorded before it
  std::function<void()> next_round;    // the solve's next round, first half, queued while the host waits
  double gap_ms = 0.0;
  long long reuse_token = 0;      // set by emst_context_reuse_tree: the next building block may skip its build
  bool state_on_device = false;   // building-block arrays are device pointers (emst_context_set_state_on_device)
  // find_component_outgoing_edges keeps its nearest-foreign proofs for the next call on the
  // same tree when that call's components coarsen these (foreign sets only shrink then)
  DevBuf<float> bb_nfn;           // the proofs (slot order)
  DevBuf<int> bb_prev;            // the labels they were proved under
  DevBuf<unsigned> ident;         // identity permutation (the merge building block: point order is slot order)
  long long ident_n = 0;
  long long bb_token = 0;         // tree they belong to (0: none)
  double bb_skip = 0.0;           // share of the last call's queries settled up front
  int bb_calls = 0;               // calls so far in the chain of coarsening calls (the solve's round - 1)
};

namespace {

template <class K, class... A>
void launch(emst_context* c, K kernel, unsigned grid, unsigned block, size_t smem, A... args) {
  kernel<<<grid, block, smem, c->stream>>>(args...);
  c->launches++;
  CK(cudaGetLastError());
}

long long* dev_counter(emst_context* c, int i) { return c->counters.p + i; }

cudaEvent_t timer_event(emst_context* c) {
  if (c->ev_next == c->ev_pool.size()) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    c->ev_pool.push_back(e);
  }
  cudaEvent_t e = c->ev_pool[c->ev_next++];
  CK(cudaEventRecord(e, c->stream));
  return e;
}

// Collect the first `upto` recorded timers (all of them by default; their events
// are complete).  The event pool is recycled only once no timer is pending.
void timers_resolve(emst_context* c, size_t upto = (size_t)-1) {
  upto = std::min(upto, c->timers.size());
  for (size_t i = 0; i < upto; ++i) {
    const auto& t = c->timers[i];
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, t.a, t.b));
    if (t.acc) *t.acc += ms;
    if (t.trav) {
      c->traverse_ms += ms;
      if (c->trace) fprintf(stderr, "[emst] round %d traverse [%lld, %lld): %.3f ms\n", t.round, t.q0, t.q1, ms);
    }
  }
  c->timers.erase(c->timers.begin(), c->timers.begin() + (long)upto);
  if (c->timers.empty()) c->ev_next = 0;
}
// The counters read in two halves: queue the copy (and note the timers it
// covers), then, after more work has been queued behind it, wait for it.
void read_counters_async(emst_context* c) {
  CK(cudaMemcpyAsync(c->host_counters, c->counters.p, kCounters * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
  if (!c->ev_counters) CK(cudaEventCreateWithFlags(&c->ev_counters, cudaEventDisableTiming));
  CK(cudaEventRecord(c->ev_counters, c->stream));
  c->counters_timers = c->timers.size();
}
void read_counters_finish(emst_context* c) {
  CK(cudaEventSynchronize(c->ev_counters));
  timers_resolve(c, c->counters_timers);
  if (c->front_pending) {   // the labelling kernel's count of nodes still mixed
    c->front_n = (long long)(unsigned)c->host_counters[8];
    c->front_pending = false;
    if (c->trace) fprintf(stderr, "[emst] comps %lld: %lld nodes still mixed\n", c->round_comps, c->front_n);
  }
}
void read_counters(emst_context* c) {
  read_counters_async(c);
  read_counters_finish(c);
}

// ------------------------------------------------------------------- scan
template <class Op>
void run_scan(emst_context* c, long long n, Op op, bool want_total) {
  // one resident block per segment: grid bounded by the occupancy
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_scan<Op>, kScanThreads, 0));
  const long long max_blocks = (long long)c->num_sms * std::max(per_sm, 1);
  const long long tiles = std::max<long long>(1, scan_tiles(n));
  const long long tiles_per_seg = (tiles + max_blocks - 1) / max_blocks;
  const long long seg = tiles_per_seg * kScanTile;
  const long long blocks = std::max<long long>(1, (n + seg - 1) / seg);
  c->scan_scratch.ensure(blocks);
  CK(cudaMemsetAsync(c->scan_scratch.p, 0, blocks * sizeof(unsigned long long), c->stream));
  unsigned long long* total = reinterpret_cast<unsigned long long*>(dev_counter(c, 1));
  launch(c, k_scan<Op>, (unsigned)blocks, kScanThreads, 0, n, seg, c->scan_scratch.p, op,
         want_total ? total : (unsigned long long*)nullptr);
}

// ------------------------------------------------------------------- sort
__global__ void k_iota_u32(unsigned* a, long long n) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) a[i] = (unsigned)i;
}

template <class K, int O, bool I>
void sort_pass(emst_context* c, long long n, const K* kin, const unsigned* vin, void* kout, unsigned* vout, int shift,
               int p, int slot) {
  auto kern = k_onesweep<K, O, I>;
  const size_t smem = sizeof(SortSmemT<K>);
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));   // (host-side, cheap)
  const long long tiles = sort_tiles(n);
  CK(cudaMemsetAsync(c->sort_status.p, 0, (size_t)tiles * kRadix * sizeof(unsigned), c->stream));
  launch(c, kern, (unsigned)tiles, kSortThreads, smem, kin, vin,
         reinterpret_cast<typename SortOutKey<K, O>::type*>(kout), vout, n, shift,
         (const unsigned*)(c->sort_off.p + p * kRadix), c->sort_status.p, c->sort_misc.p + 1 + slot);
}

template <class K, int O>
void sort_pass_v(emst_context* c, long long n, const K* kin, const unsigned* vin, bool iota, void* kout,
                 unsigned* vout, int shift, int p, int slot) {
  if (iota) sort_pass<K, O, true>(c, n, kin, nullptr, kout, vout, shift, p, slot);
  else sort_pass<K, O, false>(c, n, kin, vin, kout, vout, shift, p, slot);
}

// Histograms of the first `passes` 8-bit digits of n keys and their exclusive
// offsets; bit p of sort_misc[0] is set when digit p varies (a pass over it is
// not the identity).  No host sync.
template <class K>
void sort_prepare(emst_context* c, long long n, int passes, const K* keys) {
  c->sort_hist.ensure(kMaxPasses * kRadix);
  c->sort_off.ensure(kMaxPasses * kRadix);
  c->sort_misc.ensure(16);
  c->sort_status.ensure((size_t)sort_tiles(n) * kRadix);
  CK(cudaMemsetAsync(c->sort_hist.p, 0, kMaxPasses * kRadix * sizeof(unsigned), c->stream));
  CK(cudaMemsetAsync(c->sort_misc.p, 0, 16 * sizeof(unsigned), c->stream));
  launch(c, k_digit_histograms<K>, (unsigned)std::min<long long>(grid_for(n, kSortThreads), (long long)c->num_sms * 4),
         kSortThreads, 0, keys, n, passes, c->sort_hist.p);
  launch(c, k_digit_offsets, (unsigned)passes, kRadix, 0, (const unsigned*)c->sort_hist.p, n, c->sort_off.p,
         c->sort_misc.p);
}

// Stable LSD sort of u64 keys with the identity as values, over the digits set
// in `active` (from sort_prepare): the permutation only (bvh.py:317 -- the
// sorted keys are not written back; k_gather recomputes them).  While the low
// digits are sorted the whole key travels; once only digits >= 4 remain, only
// its high 32 bits do, and the last pass writes just the values (24 -> 16 -> 8
// bytes per key written).  Ping-pongs between k0/k1 and v0/v1; returns the buffer
// holding the permutation.
unsigned* sort_permutation(emst_context* c, long long n, unsigned long long* keys, unsigned active) {
  std::vector<int> act;
  for (int p = 0; p < kMaxPasses; ++p)
    if (active & (1u << p)) act.push_back(p);
  if (act.empty()) {   // every digit constant: the identity
    launch(c, k_iota_u32, grid_for(n, 256), 256, 0, c->v0.p, n);
    return c->v0.p;
  }
  void* kin = const_cast<unsigned long long*>(keys);
  void* kout = (void*)keys == (void*)c->k0.p ? (void*)c->k1.p : (void*)c->k0.p;
  unsigned *vin = c->v0.p, *vout = c->v1.p;
  bool wide = true, iota = true;
  for (size_t i = 0; i < act.size(); ++i) {
    const int p = act[i];
    const bool last = i + 1 == act.size();
    const int out = last ? kOutNone : (wide && act[i + 1] >= 4) ? kOutHigh32 : kOutSame;
    if (wide) {
      const auto* k = reinterpret_cast<const unsigned long long*>(kin);
      if (out == kOutNone) sort_pass_v<unsigned long long, kOutNone>(c, n, k, vin, iota, kout, vout, p * 8, p, (int)i);
      else if (out == kOutHigh32) sort_pass_v<unsigned long long, kOutHigh32>(c, n, k, vin, iota, kout, vout, p * 8, p, (int)i);
      else sort_pass_v<unsigned long long, kOutSame>(c, n, k, vin, iota, kout, vout, p * 8, p, (int)i);
    } else {
      const auto* k = reinterpret_cast<const unsigned*>(kin);
      if (out == kOutNone) sort_pass_v<unsigned, kOutNone>(c, n, k, vin, iota, kout, vout, p * 8 - 32, p, (int)i);
      else sort_pass_v<unsigned, kOutSame>(c, n, k, vin, iota, kout, vout, p * 8 - 32, p, (int)i);
    }
    if (out == kOutHigh32) wide = false;
    iota = false;
    // the next pass reads what this one wrote; its input (the codes, at first) is free
    std::swap(kin, kout);
    std::swap(vin, vout);
  }
  return vin;
}

// Stable sort of (keys, vals) by the low `bits` key bits (general u64 form:
// the building blocks and the final order's long-tie fallback).  `iota` means
// vals is the identity permutation (not read; generated in the first pass).
// keys_alt / vals_alt are the ping-pong partners; *keys_res / *vals_res receive
// whichever pair holds the result.  Reads the active-digit mask back (a sync).
void radix_sort(emst_context* c, long long n, int bits, unsigned long long* keys, unsigned* vals, bool iota,
                unsigned long long* keys_alt, unsigned* vals_alt, unsigned long long** keys_res, unsigned** vals_res) {
  const int passes = (bits + kRadixBits - 1) / kRadixBits;
  sort_prepare<unsigned long long>(c, n, passes, keys);
  unsigned active = 0;
  CK(cudaMemcpyAsync(&active, c->sort_misc.p, sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  unsigned long long *kin = keys, *kout = keys_alt;
  unsigned *vin = vals, *vout = vals_alt;
  int launched = 0;
  for (int p = 0; p < passes; ++p) {
    if (!(active & (1u << p))) continue;
    sort_pass_v<unsigned long long, kOutSame>(c, n, kin, vin, iota, kout, vout, p * kRadixBits, p, launched);
    iota = false;
    std::swap(kin, kout);
    std::swap(vin, vout);
    ++launched;
  }
  if (iota) launch(c, k_iota_u32, grid_for(n, 256), 256, 0, vin, n);   // every pass was the identity
  *keys_res = kin;
  *vals_res = vin;
}

// ------------------------------------------------------------------ build
void ensure_build(emst_context* c, long long n, int d) {
  const size_t node_bytes = d == 3 ? sizeof(Node3) : sizeof(Node2);
  c->pts.ensure((size_t)n * d);
  c->scene.ensure(1);
  c->part_lo.ensure((size_t)c->num_sms * 8 * 3);
  c->part_hi.ensure((size_t)c->num_sms * 8 * 3);
  c->part_bad.ensure((size_t)c->num_sms * 8);
  c->k0.ensure(n);
  c->k1.ensure(n);
  c->v0.ensure(n);
  c->v1.ensure(n);
  c->spts.ensure(n);
  c->perm.ensure(n);
  c->iperm.ensure(n);
  c->nodes.ensure((size_t)std::max<long long>(n - 1, 1) * node_bytes);
  c->range.ensure(std::max<long long>(n - 1, 1));
  c->node_parent.ensure(std::max<long long>(n - 1, 1));
  c->leaf_parent.ensure(n);
  c->node_delta.ensure(std::max<long long>(n - 1, 1));
  c->up.ensure(std::max<long long>(n - 1, 1));
  c->arrivals.ensure(std::max<long long>(n - 1, 1));
  c->root_box.ensure(1);
  c->counters.ensure(kCounters);
  c->nodes_stride = node_bytes;
}

// Validates and builds the hierarchy; the points must already be in c->pts
// (or at `dev_pts`).  Returns after a sync with the scene checked.
void build_tree(emst_context* c, const float* dev_pts, long long n, int d) {
  ensure_build(c, n, d);
  c->tree_valid = false;
  c->dim = d;
  c->n = n;
  CK(cudaMemsetAsync(c->scene.p, 0, sizeof(Scene), c->stream));
  unsigned sg = (unsigned)std::min<long long>(grid_for(n, kSceneThreads), (long long)c->num_sms * 8);
  if (d == 3)
    launch(c, k_scene<3>, sg, kSceneThreads, 0, dev_pts, n, c->part_lo.p, c->part_hi.p, c->part_bad.p, c->scene.p);
  else
    launch(c, k_scene<2>, sg, kSceneThreads, 0, dev_pts, n, c->part_lo.p, c->part_hi.p, c->part_bad.p, c->scene.p);
  if (d == 3) launch(c, k_morton<3>, grid_for(n, 256), 256, 0, dev_pts, n, (const Scene*)c->scene.p, c->k0.p);
  else launch(c, k_morton<2>, grid_for(n, 256), 256, 0, dev_pts, n, (const Scene*)c->scene.p, c->k0.p);
  // digit histograms of the codes; the scene check needs the host anyway, so the
  // mask of varying digits comes back with it (the build's one sync)
  sort_prepare<unsigned long long>(c, n, kMaxPasses, c->k0.p);
  Scene sc;
  unsigned active = 0;
  CK(cudaMemcpyAsync(&sc, c->scene.p, sizeof(Scene), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(&active, c->sort_misc.p, sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (sc.bad_row != 0x7fffffffffffffffll) {
    Failure f;
    f.code = EMST_ERR_NONFINITE;
    snprintf(f.msg, sizeof(f.msg), "point %lld has a non-finite coordinate", sc.bad_row);
    throw f;
  }
  unsigned* svals = sort_permutation(c, n, c->k0.p, active);
  // slot-order points, perm / iperm, and the sorted codes (recomputed) into k0
  unsigned long long* skeys = c->k0.p;
  {
    const unsigned g = grid_for(n, kGatherThreads * kGatherPer);
    // the inverse permutation: in the gather for small n, else by parts of <= kIpermPart targets
    const int parts = c->iperm_parts > 0 ? c->iperm_parts : (int)((n + kIpermPart - 1) / kIpermPart);
    unsigned* ip = parts <= 1 ? c->iperm.p : nullptr;
    if (d == 3)
      launch(c, k_gather<3>, g, kGatherThreads, 0, dev_pts, n, (const unsigned*)svals, c->perm.p, c->spts.p, ip,
             (const Scene*)c->scene.p, skeys);
    else
      launch(c, k_gather<2>, g, kGatherThreads, 0, dev_pts, n, (const unsigned*)svals, c->perm.p, c->spts.p, ip,
             (const Scene*)c->scene.p, skeys);
    if (!ip) {
      for (int k = 0; k < parts; ++k) {
        const unsigned lo = (unsigned)(k * n / parts), hi = (unsigned)((k + 1) * n / parts);
        launch(c, k_inverse_perm, (unsigned)c->num_sms * 8, 256, 0, (const unsigned*)c->perm.p, n, lo, hi, c->iperm.p);
      }
    }
  }
  if (n > 1) {
    const long long m = n - 1;
    CK(cudaMemsetAsync(c->arrivals.p, 0, m * sizeof(unsigned), c->stream));
    unsigned* up_n = reinterpret_cast<unsigned*>(dev_counter(c, 15));
    CK(cudaMemsetAsync(up_n, 0, sizeof(long long), c->stream));
    int* up_list = reinterpret_cast<int*>(c->v0.p);   // (the sort's value buffer is free after the gather)
    const unsigned up_grid = (unsigned)c->num_sms * 8;
    if (d == 3) {
      Node3* nodes = reinterpret_cast<Node3*>(c->nodes.p);
      launch(c, k_karras<Node3>, grid_for(m, 256), 256, 0, (const unsigned long long*)skeys, n, nodes, c->range.p,
             c->node_parent.p, c->leaf_parent.p, c->node_delta.p);
      CK(cudaFuncSetAttribute(k_refit<Node3, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)refit_smem<3>()));
      launch(c, k_refit<Node3, 3>, grid_for(n, kRefitThreads), kRefitThreads, refit_smem<3>(), (const float4*)c->spts.p, n, nodes,
             (const int2*)c->range.p,
             (const int*)c->node_parent.p, (const int*)c->leaf_parent.p, c->arrivals.p, c->root_box.p, up_list, up_n);
      launch(c, k_refit_up<Node3>, up_grid, 256, 0, nodes, (const int*)c->node_parent.p, c->arrivals.p,
             (const int*)up_list, (const unsigned*)up_n, c->root_box.p);
    } else {
      Node2* nodes = reinterpret_cast<Node2*>(c->nodes.p);
      launch(c, k_karras<Node2>, grid_for(m, 256), 256, 0, (const unsigned long long*)skeys, n, nodes, c->range.p,
             c->node_parent.p, c->leaf_parent.p, c->node_delta.p);
      CK(cudaFuncSetAttribute(k_refit<Node2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)refit_smem<2>()));
      launch(c, k_refit<Node2, 2>, grid_for(n, kRefitThreads), kRefitThreads, refit_smem<2>(), (const float4*)c->spts.p, n, nodes,
             (const int2*)c->range.p,
             (const int*)c->node_parent.p, (const int*)c->leaf_parent.p, c->arrivals.p, c->root_box.p, up_list, up_n);
      launch(c, k_refit_up<Node2>, up_grid, 256, 0, nodes, (const int*)c->node_parent.p, c->arrivals.p,
             (const int*)up_list, (const unsigned*)up_n, c->root_box.p);
    }
  }
  if (n > 1)
    launch(c, k_pack_up, grid_for(n - 1, 256), 256, 0, (const int*)c->node_parent.p, (const int*)c->node_delta.p, n - 1,
           c->up.p);
  c->tree_valid = true;
  c->tree_token++;
}

const float* stage_points(emst_context* c, const float* pts, long long n, int d, int flags, emst_stats* st) {
  if (flags & EMST_POINTS_ON_DEVICE) return pts;
  c->pts.ensure((size_t)n * d);
  const size_t bytes = (size_t)n * d * sizeof(float);
  const auto t0 = std::chrono::steady_clock::now();
  if (c->staging && bytes >= (4u << 20) && !emst_host::is_pinned(pts)) {
    CK(c->stager.init());
    CK(c->stager.h2d(c->pts.p, pts, bytes, c->stream));
  } else {
    CK(cudaMemcpyAsync(c->pts.p, pts, bytes, cudaMemcpyHostToDevice, c->stream));
  }
  if (st) st->host_in_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (st) st->h2d_bytes += (long long)n * d * sizeof(float);
  return c->pts.p;
}

void check_shape(long long n, int d) {
  if (n <= 0) fail(EMST_ERR_EMPTY, "point set is empty");
  if (d != 2 && d != 3) fail(EMST_ERR_DIM, "points must have 2 or 3 coordinates, got %d", d);
  if (n >= (1ll << 30)) fail(EMST_ERR_TOO_LARGE, "n = %lld exceeds the 2^30 - 1 point limit", n);
}

// ----------------------------------------------------------------- rounds
void ensure_rounds(emst_context* c, long long n) {
  c->label.ensure(n);
  c->bprefix.ensure(n);
  c->nfn_lb.ensure(n);
  c->big_tops.ensure(n / kDirectFill + n / kFillChunk + 2);   // top pure ranges are disjoint
  c->front[0].ensure(std::max<long long>(n - 1, 1));
  c->front[1].ensure(std::max<long long>(n - 1, 1));
  c->top.ensure(n);
  c->ub.ensure(n);
  c->best.ensure(n);
  c->succ.ensure(n);
  c->ptr.ensure(n);
  c->root.ensure(n);
  c->newid.ensure(n);
  c->fin.ensure(n);
  c->eout.ensure(n);
}

__global__ void k_iota_int(int* a, long long n) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) a[i] = (int)i;
}

// node labels + upper bounds for the current labels (phases 1-2 of a round)
// Node labelling modes for round_prepare
enum LabelMode {
  kLabelsFull,       // every node, reference semantics (building blocks, subtree_skip off)
  kLabelsNone,       // round 1: every child label is still the build's MIXED, and a
                     // query never reaches its own leaf, so nothing to write
  kLabelsFrontier,   // only the nodes that were mixed last round (see k_node_labels_front)
};

template <class Node>
void launch_labels(emst_context* c, long long n, LabelMode mode, bool want_top) {
  const long long m = n - 1;
  Node* nodes = reinterpret_cast<Node*>(c->nodes.p);
  if (mode == kLabelsFull) {
    launch(c, k_node_labels<Node>, grid_for(m, 256), 256, 0, nodes, (const int2*)c->range.p, (const int*)c->bprefix.p,
           (const int*)c->label.p, m);
    return;
  }
  unsigned* big_n = reinterpret_cast<unsigned*>(dev_counter(c, 10));
  CK(cudaMemsetAsync(big_n, 0, sizeof(long long), c->stream));
  const long long count = c->front_n < 0 ? m : c->front_n;
  const int* in = c->front_n < 0 ? nullptr : c->front[c->front_cur].p;
  int* out = c->front[c->front_cur ^ 1].p;
  unsigned* out_n = reinterpret_cast<unsigned*>(dev_counter(c, 8));
  CK(cudaMemsetAsync(out_n, 0, sizeof(long long), c->stream));
  if (count > 0)
    launch(c, k_node_labels_front<Node>, grid_for(count, kLabelThreads), kLabelThreads, 0, nodes, (const int2*)c->range.p,
           (const int*)c->bprefix.p, (const int*)c->label.p, in, count, out, out_n,
           want_top ? c->top.p : (int*)nullptr, c->big_tops.p, big_n);
  if (want_top)
    launch(c, k_fill_top, (unsigned)c->num_sms * 8, 256, 0, (const int4*)c->big_tops.p,
           (const unsigned*)big_n, c->top.p);
  c->front_cur ^= 1;
  c->front_pending = true;   // front_n is read back with the round's counters
}

void allreduce_u64(emst_context* c, unsigned long long* buf, long long count, int rows, long long stride, bool sum);

// Phase 1 of a round, first half: the component bounds (boundary-pair and window
// seeds) and the boundary prefix the labels need.  Uses the labels, c->round and
// c->round_comps (an upper bound is enough: it only steers the window seeds).
void prepare_bounds(emst_context* c, long long n, bool bounds, double* ms_bounds, LabelMode mode) {
  if (c->trace && c->merge_end && c->round > 1) {
    // (trace) the device's idle time from the last merge to this round's first kernel
    CK(cudaEventSynchronize(c->merge_end));
    cudaEvent_t now = timer_event(c);
    CK(cudaEventSynchronize(now));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->merge_end, now));
    c->gap_ms += ms;
  }
  // Ranks of a multi-GPU solve (rounds >= 2) seed the bounds of their own Morton range only and
  // meet in one min-allreduce; round 1's streaming seeds and the building blocks stay replicated.
  const bool sharded = bounds && c->world > 1 && c->round > 1;
  const long long r0 = sharded ? c->rank * n / c->world : 0, r1 = sharded ? (c->rank + 1) * n / c->world : n;
  // window seeds pay while components are small and in 3D (measured: 37M blobs 3D
  // -2.3 ms, 10M normal 3D -0.6 ms; the 2D configs lose ~1 %); later rounds gain nothing
  // (±8 in 3D, ±4 in 2D: 24M blobs 2D 29.9 -> 29.65 ms, 10M uniform 2D 13.65 -> 13.6; ±8 and ±2 less)
  const int seed_w = c->dim == 3 ? c->seed_window : c->seed_window_2d;
  const bool window = bounds && seed_w > 1 && c->round >= c->seed_from && !c->core && c->round_comps * 1024 >= n;
  cudaEvent_t e0 = timer_event(c);
  if (mode == kLabelsNone && c->round == 1) {
    // round 1 of the solve: singletons, no node labels, so no boundary prefix either
    if (bounds) {
      // Euclidean round 1: each slot's nearest of its Z-neighbours +-8 (measured +-1 / 2 / 4 / 8 / 16 /
      // 24 at 37M blobs 3D: 67.05 / - / - / 66.72 / 66.86 / 67.17 ms; round 1 9.07 -> 8.40 ms at +-8)
      if (!c->core) {
        if (c->dim == 3) launch(c, k_seed_round1_window<3, EMST_SEED1_W>, grid_for(n, kSeed1Threads), kSeed1Threads, 0, (const float4*)c->spts.p, n, c->ub.p);
        else launch(c, k_seed_round1_window<2, EMST_SEED1_W>, grid_for(n, kSeed1Threads), kSeed1Threads, 0, (const float4*)c->spts.p, n, c->ub.p);
      } else if (c->dim == 3) launch(c, k_seed_round1<3>, grid_for(n, 256), 256, 0, (const float4*)c->spts.p, n, c->core, c->ub.p);
      else launch(c, k_seed_round1<2>, grid_for(n, 256), 256, 0, (const float4*)c->spts.p, n, c->core, c->ub.p);
    }
  } else {
    // ranks of a multi-GPU solve seed only the boundary pairs of their own Morton range [r0, r1)
    // (exact weights for the building block compute_upper_bounds, round 0; upper bounds in the solve)
    // (the window's pairs include every boundary pair (s, s + 1): with the window on, the
    // scan only counts the boundaries)
    run_scan(c, n, RoundScanOp{c->label.p, c->spts.p, c->ub.p, c->bprefix.p, n, c->dim, bounds && !window, c->core,
                               c->round == 0, r0, r1},
             false);
  }
  if (window) {
    const int W = std::min(seed_w, kSeedMaxW);
    const auto kern = c->dim == 3 ? (W == 8 ? k_seed_window<3, 8> : k_seed_window<3, 0>)
                                  : (W == 4 ? k_seed_window<2, 4> : k_seed_window<2, 0>);
    const long long b0 = r0 / kSeedThreads, b1 = (r1 + kSeedThreads - 1) / kSeedThreads;   // blocks covering [r0, r1)
    launch(c, kern, (unsigned)std::max<long long>(1, b1 - b0), kSeedThreads, 0, (const int*)c->label.p,
           (const float4*)c->spts.p, n, W, c->ub.p, b0);
  }
  c->timers.push_back({e0, timer_event(c), ms_bounds, false, c->round, 0, 0});
}

// The ranks' seeds meet in one min-allreduce of the c bounds (u64 bit patterns); needs
// the exact component count.
void exchange_bounds(emst_context* c, bool bounds, double* ms_bounds) {
  if (!(bounds && c->world > 1 && c->round > 1)) return;
  cudaEvent_t e0 = timer_event(c);
  allreduce_u64(c, c->ub.p, c->round_comps, 1, 0, false);
  c->timers.push_back({e0, timer_event(c), ms_bounds, false, c->round, 0, 0});
}

// Phase 1, second half: the node labels (needs the last labelling's count of mixed nodes).
void prepare_labels(emst_context* c, long long n, double* ms_labels, bool want_top, LabelMode mode) {
  c->top_valid = false;
  cudaEvent_t e1 = timer_event(c);
  if (n > 1 && mode != kLabelsNone) {
    if (c->dim == 3) launch_labels<Node3>(c, n, mode, want_top);
    else launch_labels<Node2>(c, n, mode, want_top);
    c->top_valid = want_top && mode == kLabelsFrontier;
  }
  // (no sync here: the times and the count of nodes still mixed are read at the round's counter read)
  c->timers.push_back({e1, timer_event(c), ms_labels, false, c->round, 0, 0});
}

void round_prepare(emst_context* c, long long n, bool bounds, double* ms_labels, double* ms_bounds,
                   bool want_top = false, LabelMode mode = kLabelsFull) {
  prepare_bounds(c, n, bounds, ms_bounds, mode);
  exchange_bounds(c, bounds, ms_bounds);
  prepare_labels(c, n, ms_labels, want_top, mode);
}

template <int D, bool S, bool B, bool M, bool P, bool G = false>
void traverse_range_m(emst_context* c, EdgeKey* out, long long q0, long long q1) {
  if (q1 <= q0) return;
  using Node = typename NodeOf<D>::type;
  auto kernel = k_traverse<D, S, B, M, P, G>;
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kTraverseThreads, 0));
  // Small launches (fewer queries than two per resident lane) claim half chunks, so that more
  // warps start at once: there each query's chain of L2 round trips, not throughput, is the time
  // (listed rounds: the list is about the share of queries the last round did not settle up front)
  const bool listed = P && B && !M && c->round > 1 && c->skip_frac >= c->list_skip;
  const double expect = listed ? std::max(0.0, 1.0 - c->skip_frac) * (double)(q1 - q0) : (double)(q1 - q0);
  const long long resident_warps = (long long)c->num_sms * std::max(per_sm, 1) * (kTraverseThreads / 32);
#ifdef EMST_CLAIM_FIXED
  const int claim = kTraverseChunk;   // (A/B build)
  (void)expect;
  (void)resident_warps;
#else
  const int claim = expect <= (double)(resident_warps * kTraverseChunk) ? kTraverseChunk / 2 : kTraverseChunk;
#endif
  const long long warps_needed = (q1 - q0 + claim - 1) / claim;
  const long long blocks_needed = (warps_needed + kTraverseThreads / 32 - 1) / (kTraverseThreads / 32);
  const unsigned grid = (unsigned)std::max<long long>(1, std::min<long long>((long long)c->num_sms * std::max(per_sm, 1),
                                                                             blocks_needed));
  unsigned long long* work = reinterpret_cast<unsigned long long*>(dev_counter(c, 4));
  CK(cudaMemsetAsync(work, 0, sizeof(unsigned long long), c->stream));
  const int* side = c->one_side && P ? (const int*)dev_counter(c, 13) : (const int*)nullptr;
  // late rounds: list the queries that are not settled up front (Euclidean with bounds only)
  const bool use_list = P && B && !M && c->round > 1 && c->skip_frac >= c->list_skip;
  unsigned* qcount = reinterpret_cast<unsigned*>(dev_counter(c, 14));
  cudaEvent_t ta = timer_event(c);
  if (use_list) {
    c->qlist.ensure(q1 - q0);
    CK(cudaMemsetAsync(qcount, 0, sizeof(long long), c->stream));
    static int pf_per_sm[4] = {0, 0, 0, 0};   // resident blocks per SM (one wave, no tail)
    if (!pf_per_sm[D]) CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pf_per_sm[D], k_prefilter<D>, kScanThreads, 0));
    const unsigned pg = (unsigned)std::min<long long>(grid_for(q1 - q0, kScanTile),
                                                      (long long)c->num_sms * std::max(pf_per_sm[D], 1));
    launch(c, k_prefilter<D>, pg, kScanThreads, 0, (const float4*)c->spts.p, (const int*)c->label.p,
           (const unsigned long long*)c->ub.p, (const float*)c->nfn_lb.p,
           c->top_valid ? (const int*)c->top.p : (const int*)nullptr, (const int2*)c->up.p, (const Scene*)c->scene.p,
           q0, q1, side, c->qlist.p, qcount, reinterpret_cast<unsigned long long*>(dev_counter(c, 9)));
  }
  {
    launch(c, kernel, grid, kTraverseThreads, 0, (const Node*)reinterpret_cast<Node*>(c->nodes.p),
           (const float4*)c->spts.p, (const unsigned*)c->perm.p, (const int*)c->label.p, c->ub.p, out, q0, q1,
           (const Box3*)c->root_box.p, reinterpret_cast<unsigned long long*>(dev_counter(c, 0)),
           reinterpret_cast<int*>(dev_counter(c, 3)), work, c->singleton_round && c->vshards == 1 && c->world == 1,
           c->nfn_lb.p, (const int2*)c->up.p, (const int*)c->leaf_parent.p, (const Scene*)c->scene.p,
           c->top_valid ? (const int*)c->top.p : (const int*)nullptr, c->core, side,
           use_list ? (const int*)c->qlist.p : (const int*)nullptr, (const unsigned*)qcount, claim);
  }
  c->timers.push_back({ta, timer_event(c), nullptr, true, c->round, q0, q1});   // traverse_ms at the next sync
  c->traverse_launches++;
  c->traverse_queries += q1 - q0;
}

template <int D, bool S, bool B>
void traverse_range(emst_context* c, EdgeKey* out, long long q0, long long q1) {
  const bool single = c->singleton_round && c->vshards == 1 && c->world == 1;
  if (c->core) traverse_range_m<D, S, B, true, false>(c, out, q0, q1);
  else if (single && c->single_kernel) traverse_range_m<D, S, B, false, false, true>(c, out, q0, q1);
  else if (B && c->round >= c->proof_from && c->proof_from > 0) traverse_range_m<D, S, B, false, B>(c, out, q0, q1);
  else traverse_range_m<D, S, B, false, false>(c, out, q0, q1);
}

void traverse_dispatch(emst_context* c, int flags, EdgeKey* out, long long q0, long long q1) {
  const bool S = flags & EMST_SUBTREE_SKIP, B = flags & EMST_UPPER_BOUNDS;
  if (c->dim == 3) {
    if (S && B) traverse_range<3, true, true>(c, out, q0, q1);
    else if (S) traverse_range<3, true, false>(c, out, q0, q1);
    else if (B) traverse_range<3, false, true>(c, out, q0, q1);
    else traverse_range<3, false, false>(c, out, q0, q1);
  } else {
    if (S && B) traverse_range<2, true, true>(c, out, q0, q1);
    else if (S) traverse_range<2, true, false>(c, out, q0, q1);
    else if (B) traverse_range<2, false, true>(c, out, q0, q1);
    else traverse_range<2, false, false>(c, out, q0, q1);
  }
}

// Phase 3: per-component minimum outgoing edge into c->best[0, comps).
// With two components left, both minima are the same edge (the lightest of the
// edges between them under (w, u, v)), so only the smaller component's queries
// run and its key is copied to the other (c->one_side).
void round_find_all(emst_context* c, long long n, long long comps, int flags);
void round_find(emst_context* c, long long n, long long comps, int flags) {
  round_find_all(c, n, comps, flags);
  // (only the proof kernels leave a side out; after the others the copy rewrites the same edge)
  if (c->one_side) launch(c, k_copy_key, 1, 32, 0, c->best.p, (const int*)dev_counter(c, 13));
}
// All-reduce-min (or sum) of `count` u64 over the local virtual shards (rows
// 0..rows-1 of `buf`, `stride` apart) and then over the ranks, result in row 0.
// The rank step is ncclAllReduce on the context's communicator (a 1-rank one
// under virtual shards, so the NCCL call path runs on a single GPU too), or
// the caller's host exchange callback (any torch.distributed backend).
void allreduce_u64(emst_context* c, unsigned long long* buf, long long count, int rows, long long stride, bool sum) {
  if (count <= 0) return;
  if (rows > 1)
    launch(c, k_fold_rows, grid_for(count, 256), 256, 0, buf, rows, stride, count, sum);
  if (c->comm) {
    NK(ncclAllReduce(buf, buf, count, ncclUint64, sum ? ncclSum : ncclMin, c->comm, c->stream));
  } else if (c->world > 1) {
    if (!c->exch_fn) fail(EMST_ERR_PARAM, "world %d context has neither an NCCL communicator nor an exchange", c->world);
    c->exch_host.ensure_host(count);
    CK(cudaMemcpyAsync(c->exch_host.p, buf, count * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (c->exch_fn(reinterpret_cast<uint64_t*>(c->exch_host.p), count, sum ? EMST_EXCHANGE_SUM : EMST_EXCHANGE_MIN,
                   c->exch_user) != 0)
      fail(EMST_ERR_NCCL, "host exchange callback failed");
    CK(cudaMemcpyAsync(buf, c->exch_host.p, count * sizeof(unsigned long long), cudaMemcpyHostToDevice, c->stream));
  }
}

// Per-component minimum over all shards of the round's queries.  A shard is
// one Morton slot range [g n / S, (g + 1) n / S) of S = world * vshards; this
// rank runs its vshards ranges.  With S > 1 the keys meet in the two-phase
// exchange: min of the weight bits, then min of (u << 32 | v)
// over the shards whose weight equals it -- exact for the 128-bit (w, u, v)
// order, which no single u64 reduction is.
void round_find_all(emst_context* c, long long n, long long comps, int flags) {
  const int V = c->vshards;
  const long long S = (long long)c->world * V;
  if (S == 1) {
    traverse_dispatch(c, flags, c->best.p, 0, n);
    return;
  }
  EdgeKey* keys = c->best.p;
  if (V > 1) {
    c->shard_keys.ensure((size_t)V * comps);
    CK(cudaMemsetAsync(c->shard_keys.p, 0xff, (size_t)V * comps * sizeof(EdgeKey), c->stream));
    keys = c->shard_keys.p;
  }
  for (int g = 0; g < V; ++g) {
    const long long s = (long long)c->rank * V + g;
    traverse_dispatch(c, flags, keys + (size_t)g * comps, s * n / S, (s + 1) * n / S);
  }
  c->xw.ensure((size_t)V * comps);
  c->xuv.ensure((size_t)V * comps);
  for (int g = 0; g < V; ++g)
    launch(c, k_split_keys, grid_for(comps, 256), 256, 0, (const EdgeKey*)(keys + (size_t)g * comps), comps,
           c->xw.p + (size_t)g * comps);
  allreduce_u64(c, c->xw.p, comps, V, comps, false);
  for (int g = 0; g < V; ++g)
    launch(c, k_mask_uv, grid_for(comps, 256), 256, 0, (const EdgeKey*)(keys + (size_t)g * comps),
           (const unsigned long long*)c->xw.p, comps, c->xuv.p + (size_t)g * comps);
  allreduce_u64(c, c->xuv.p, comps, V, comps, false);
  launch(c, k_join_keys, grid_for(comps, 256), 256, 0, c->best.p, (const unsigned long long*)c->xw.p,
         (const unsigned long long*)c->xuv.p, comps);
}

// Phase 4: collapse the successor graph; appends edges at `edge_base`, relabels.
// Returns the new component count (and the edges emitted via *emitted).
// singletons: the solve's round 1, where label[s] == s
long long round_merge(emst_context* c, long long n, long long comps, long long edge_base, long long* emitted,
                      double* ms_merge = nullptr, bool singletons = false, const unsigned* iperm = nullptr) {
  // (the solve's next-round work to queue behind the counter copy; consumed here, once)
  std::function<void()> next_round = std::move(c->next_round);
  c->next_round = nullptr;
  cudaEvent_t m0 = timer_event(c);
  int* err = reinterpret_cast<int*>(dev_counter(c, 2));
  // (an explicit iperm is the identity, its own inverse)
  launch(c, k_merge_succ, grid_for(comps, 256), 256, 0, (const EdgeKey*)c->best.p, comps, (const int*)c->label.p,
         iperm ? iperm : (const unsigned*)c->perm.p, iperm ? iperm : (const unsigned*)c->iperm.p, c->succ.p, err,
         singletons);
  launch(c, k_merge_link, grid_for(comps, 256), 256, 0, (const int*)c->succ.p, comps, c->ptr.p);
  launch(c, k_merge_jump, grid_for(comps, 256), 256, 0, c->ptr.p, comps, c->root.p, err);
  // (the flag cache borrows fin, which k_merge_final writes after the scan)
  run_scan(c, comps, MergeScanOp{c->succ.p, c->root.p, c->best.p, c->eout.p, edge_base, c->newid.p,
                                 reinterpret_cast<unsigned char*>(c->fin.p)},
           true);
  launch(c, k_merge_final, grid_for(comps, 256), 256, 0, (const int*)c->root.p, (const int*)c->newid.p, comps, c->fin.p);
  launch(c, k_relabel, grid_for((n + 3) / 4, 256), 256, 0, c->label.p, (const int*)c->fin.p, n);
  c->merge_end = timer_event(c);
  c->timers.push_back({m0, c->merge_end, ms_merge, false, c->round, 0, 0});
  read_counters_async(c);
  if (next_round) next_round();   // (work queued behind the counter copy, before the host waits)
  read_counters_finish(c);   // (the round's one host sync; it also collects the round's timers)
  long long* h = c->host_counters;
  if (h[2] & kErrNoEdge) fail(EMST_ERR_NO_EDGE, "a component found no valid outgoing edge");
  if (h[2] & kErrChain) fail(EMST_ERR_CHAIN, "component chain did not terminate in a pair");
  unsigned long long tot = (unsigned long long)h[1];
  *emitted = (long long)(tot & 0x7fffffffull);
  return (long long)(tot >> 31);
}

// Final order (w, u, v) of the n - 1 edges (mst.py:745-747): a 4-pass stable
// radix sort on the f32-rounded weight (16 bytes per edge per pass instead of
// 24 over 8 passes on the f64 bits), then every run of equal keys put in exact
// (w, u, v) order (k_edge_ties and the warp / block fix-ups, which take their
// run counts from the device: no host sync).  A run longer than kBlockTie
// (checked by the caller at the solve's final counter read, sort_overflowed)
// is redone by sort_and_emit_exact.
// (key: the sorted 32-bit keys, whose two-runs the emit orders; nullptr: order is final)
void emit_edges(emst_context* c, const unsigned* order, const unsigned* key, long long ne, long long* edges_dst,
                double* w_dst, bool packed) {
  if (packed)
    launch(c, k_edge_emit_packed, grid_for(ne, 256), 256, 0, order, (const EdgeKey*)c->eout.p, key, ne,
           reinterpret_cast<unsigned long long*>(edges_dst), w_dst, 0ll, ne);
  else
    launch(c, k_edge_emit, grid_for(ne, 256), 256, 0, order, (const EdgeKey*)c->eout.p, key, ne, edges_dst, w_dst);
}

void sort_and_emit(emst_context* c, long long ne, long long* edges_dst, double* w_dst, bool packed = false,
                   bool defer_emit = false) {
  if (ne <= 0) return;
  unsigned* key = reinterpret_cast<unsigned*>(c->k0.p);
  c->sort_misc.ensure(16);
  // (min, max) of the weight bits in words 12..15 of sort_misc (reset by sort_prepare after use)
  unsigned long long* wr = reinterpret_cast<unsigned long long*>(c->sort_misc.p + 12);
  CK(cudaMemsetAsync(wr, 0xff, sizeof(unsigned long long), c->stream));
  CK(cudaMemsetAsync(wr + 1, 0, sizeof(unsigned long long), c->stream));
  launch(c, k_edge_wrange, (unsigned)std::min<long long>(grid_for(ne, 256), (long long)c->num_sms * 8), 256, 0,
         (const EdgeKey*)c->eout.p, ne, wr);
  launch(c, k_edge_wkey, grid_for(ne, 256), 256, 0, (const EdgeKey*)c->eout.p, ne, (const unsigned long long*)wr, key);
  sort_prepare<unsigned>(c, ne, 4, key);
  unsigned* kin = key;
  unsigned* kout = reinterpret_cast<unsigned*>(c->k1.p);
  unsigned *vin = c->v0.p, *vout = c->v1.p;
  for (int p = 0; p < 4; ++p) {
    sort_pass_v<unsigned, kOutSame>(c, ne, kin, vin, p == 0, kout, vout, p * 8, p, p);
    std::swap(kin, kout);
    std::swap(vin, vout);
  }
  unsigned* order = vin;
  long long* tie = dev_counter(c, 7);   // low word: longest run, high word: listed long runs
  CK(cudaMemsetAsync(tie, 0, sizeof(long long), c->stream));
  c->tie_runs.ensure(ne / (kShortTie + 1) + 1);
  unsigned* mid_n = reinterpret_cast<unsigned*>(dev_counter(c, 11));
  CK(cudaMemsetAsync(mid_n, 0, sizeof(long long), c->stream));
  c->tie_mid.ensure(ne / (kThreadTie + 1) + 1);
  c->tie_small.ensure(ne / (kShortTie + 1) + 1);
  unsigned* small_n = mid_n + 1;   // (high word of counters[11])
  launch(c, k_edge_ties, grid_for(ne, 256), 256, 0, (const unsigned*)kin, ne, (const EdgeKey*)c->eout.p, order,
         (unsigned*)tie, c->tie_runs.p, (unsigned*)tie + 1, c->tie_mid.p, mid_n, c->tie_small.p, small_n);
  // (grids sized for the worst case; the kernels stride over the device-side counts)
  launch(c, k_edge_fix_mid, (unsigned)c->num_sms * 8, 256, 0, (const int2*)c->tie_mid.p, (const unsigned*)mid_n,
         (const EdgeKey*)c->eout.p, order);
  launch(c, k_edge_fix_small, (unsigned)c->num_sms * 8, kSmallTieThreads, 0, (const int2*)c->tie_small.p,
         (const unsigned*)small_n, (const EdgeKey*)c->eout.p, order);
  CK(cudaFuncSetAttribute(k_edge_fix_long, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kEdgeFixSmem));
  launch(c, k_edge_fix_long, (unsigned)c->num_sms, 1024, kEdgeFixSmem, (const int2*)c->tie_runs.p,
         (const unsigned*)tie + 1, (const EdgeKey*)c->eout.p, order);
  if (defer_emit) {   // (the host-output path emits chunk by chunk behind its copies: emit_chunked)
    c->emit_order = order;
    c->emit_key = kin;
    return;
  }
  emit_edges(c, order, kin, ne, edges_dst, w_dst, packed);
}

// true when sort_and_emit met a tie run longer than kBlockTie (after a counter read)
bool sort_overflowed(emst_context* c) { return (unsigned)(c->host_counters[7] & 0xffffffffll) > (unsigned)kBlockTie; }

// The exact two-key order for inputs with very long runs of equal weights: a
// stable sort by (u << 32 | v), then a stable sort by the weight bits.
void sort_and_emit_exact(emst_context* c, long long ne, long long* edges_dst, double* w_dst, bool packed = false) {
  if (ne <= 0) return;
  unsigned long long* keys;
  unsigned* order;
  launch(c, k_edge_uv_keys, grid_for(ne, 256), 256, 0, (const EdgeKey*)c->eout.p, ne, c->k0.p);
  radix_sort(c, ne, 64, c->k0.p, c->v0.p, true, c->k1.p, c->v1.p, &keys, &order);
  unsigned long long* kin = keys == c->k0.p ? c->k1.p : c->k0.p;
  unsigned* vin_alt = order == c->v1.p ? c->v0.p : c->v1.p;
  launch(c, k_edge_w_keys, grid_for(ne, 256), 256, 0, (const EdgeKey*)c->eout.p, (const unsigned*)order, ne, kin);
  unsigned long long* keys2;
  unsigned* order2;
  radix_sort(c, ne, 64, kin, order, false, keys, vin_alt, &keys2, &order2);
  emit_edges(c, order2, nullptr, ne, edges_dst, w_dst, packed);
}

// float(np.sum(weights)) on the device in numpy's summation order.
void total_weight(emst_context* c, const double* w, long long ne, emst_stats* st) {
  int levels = 0;
  while (levels < kPairwiseLevels && ne >= (256ll << (levels + 1))) ++levels;
  c->pairwise.ensure(2 * (1 << kPairwiseLevels) + 1);
  double* a = c->pairwise.p;
  double* b = a + (1 << kPairwiseLevels);
  launch(c, k_pairwise_partials, grid_for(1 << levels, 128), 128, 0, w, ne, levels, a);
  // combine the recursion tree bottom-up, kCombineLevels levels per launch
  do {
    const int g = std::min(levels, kCombineLevels);
    levels -= g;
    launch(c, k_pairwise_combine, 1u << levels, 1024, 0, (const double*)a, g, b, levels == 0);
    std::swap(a, b);
  } while (levels > 0);
  CK(cudaMemcpyAsync(&st->total_weight, a, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
}

int max_iterations(long long n) {
  if (n <= 1) return 0;
  int k = 0;
  while ((1ll << k) < n) ++k;
  return std::max(k, 1);
}

// The full solve: build, rounds, final order.  Outputs land in device buffers
// c->out_edges / c->out_w unless the caller's device pointers are given.
// ------------------------------------------------------- core distances
// c->core_slot[s] = core distance of the point in slot s for k_pts (>= 2); the
// tree must be built.  The per-query heap of k_pts - 1 distances lives in shared
// memory when it fits in kCoreSmemMax bytes per block, else in global scratch.
constexpr size_t kCoreSmemMax = 96 * 1024;

template <int D>
void compute_cores_t(emst_context* c, long long n, long long k_pts) {
  using Node = typename NodeOf<D>::type;
  const int kc = (int)(k_pts - 1);
  const size_t smem = (size_t)kc * kCoreThreads * sizeof(double);
  const bool in_smem = smem <= kCoreSmemMax;
  CK(cudaFuncSetAttribute(k_core<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCoreSmemMax));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_core<D>, kCoreThreads, in_smem ? smem : 0));
  const long long blocks_needed = (n + kCoreChunk * (kCoreThreads / 32) - 1) / (kCoreChunk * (kCoreThreads / 32));
  const unsigned grid = (unsigned)std::max<long long>(1, std::min<long long>((long long)c->num_sms * std::max(per_sm, 1),
                                                                             blocks_needed));
  double* heap = nullptr;
  if (!in_smem) {
    c->core_tmp.ensure((size_t)grid * kCoreThreads * kc);
    heap = c->core_tmp.p;
  }
  unsigned long long* work = reinterpret_cast<unsigned long long*>(dev_counter(c, 4));
  CK(cudaMemsetAsync(work, 0, sizeof(unsigned long long), c->stream));
  launch(c, k_core<D>, grid, kCoreThreads, in_smem ? smem : 0, (const Node*)reinterpret_cast<Node*>(c->nodes.p),
         (const float4*)c->spts.p, 0ll, n, kc, heap, c->core_slot.p,
         reinterpret_cast<unsigned long long*>(dev_counter(c, 0)), reinterpret_cast<int*>(dev_counter(c, 3)), work,
         (const int2*)c->up.p, (const int*)c->leaf_parent.p, (const Scene*)c->scene.p);
}

// Activate mutual reachability for the current tree: core distances from a
// caller's table (original point order, host memory) or computed for k_pts.
// k_pts == 1 without a table is plain Euclidean (all cores 0, mst.py:644).
void prepare_cores(emst_context* c, long long n, long long k_pts, const double* core_host) {
  c->core = nullptr;
  if (!core_host && k_pts <= 1) return;
  c->core_slot.ensure(n);
  if (core_host) {
    c->core_tmp.ensure(n);
    CK(cudaMemcpyAsync(c->core_tmp.p, core_host, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    launch(c, k_gather_by_perm, grid_for(n, 256), 256, 0, (const double*)c->core_tmp.p, (const unsigned*)c->perm.p, n,
           c->core_slot.p);
  } else {
    if (k_pts > n) fail(EMST_ERR_PARAM, "k_pts must be in [1, %lld], got %lld", n, k_pts);
    if (c->dim == 3) compute_cores_t<3>(c, n, k_pts);
    else compute_cores_t<2>(c, n, k_pts);
    read_counters(c);
    if (c->host_counters[3]) fail(EMST_ERR_STACK, "neighbour traversal exceeded %d stacked nodes", kStackCapacity);
  }
  c->core = c->core_slot.p;
}

#ifdef EMST_VISIT_HIST
void visit_hist_reset(emst_context* c) {
  const int2* r = c->range.p;
  CK(cudaMemcpyToSymbolAsync(g_visit_range, &r, sizeof(r), 0, cudaMemcpyHostToDevice, c->stream));
  static const unsigned long long zero[2][32] = {};
  CK(cudaMemcpyToSymbolAsync(g_visit_hist, zero, sizeof(zero), 0, cudaMemcpyHostToDevice, c->stream));
}
void visit_hist_print(emst_context* c) {
  unsigned long long h[2][32];
  CK(cudaMemcpyFromSymbol(h, g_visit_hist, sizeof(h)));
  for (int k = 0; k < 2; ++k) {
    fprintf(stderr, "[emst] visits (%s) by log2 range:", k ? "pop" : "climb");
    for (int b = 0; b < 32; ++b) if (h[k][b]) fprintf(stderr, " %d:%llu", b, h[k][b]);
    fprintf(stderr, "\n");
  }
}
#endif

void solve(emst_context* c, const float* dev_pts, long long n, int d, int flags, long long* edges_dev,
           double* w_dev, emst_stats* st, long long k_pts = 1, const double* core_host = nullptr, bool packed = false) {
  cudaEvent_t t0, t1, t2, t3;
  CK(cudaEventCreate(&t0));
  CK(cudaEventCreate(&t1));
  CK(cudaEventCreate(&t2));
  CK(cudaEventCreate(&t3));
  c->timers.clear();
  c->ev_next = 0;
  CK(cudaEventRecord(t0, c->stream));
  build_tree(c, dev_pts, n, d);
  CK(cudaEventRecord(t3, c->stream));
#ifdef EMST_VISIT_HIST
  visit_hist_reset(c);
#endif
  CK(cudaMemsetAsync(c->counters.p, 0, kCounters * sizeof(long long), c->stream));
  prepare_cores(c, n, k_pts, core_host);   // (mutual reachability; the "core" phase)
  CK(cudaEventRecord(t1, c->stream));
  ensure_rounds(c, n);
  CK(cudaMemsetAsync(c->counters.p, 0, kCounters * sizeof(long long), c->stream));
  launch(c, k_iota_int, grid_for(n, 256), 256, 0, c->label.p, n);
  CK(cudaMemsetAsync(c->nfn_lb.p, 0, n * sizeof(float), c->stream));
  CK(cudaMemsetAsync(c->top.p, 0, n * sizeof(int), c->stream));
  c->front_n = -1;
  c->skip_frac = 0.0;
  c->bb_token = 0;   // (the solve reuses the round buffers)
  long long comps = n, edges = 0;
  const int max_it = max_iterations(n);
  st->component_counts[0] = n;
  st->num_counts = 1;
  double ms_labels = 0, ms_bounds = 0, ms_find = 0, ms_merge = 0;
  long long visits_before = 0, found_before = 0, skipped_before = 0;
  double tv_before = c->traverse_ms;
  const bool bounds = flags & EMST_UPPER_BOUNDS;
  const bool skip = flags & EMST_SUBTREE_SKIP;
  // A round's bounds need only the relabelled components and an upper bound of
  // their count (Boruvka at least halves it), so they are queued behind the
  // merge's counter copy: the device computes them while the host waits for
  // the counters, instead of idling between the rounds.
  bool prepped = false;   // the bounds of round st->iterations + 1 are queued
  auto queue_bounds = [&](int round, long long comps_bound, long long comps_guess) {
    CK(cudaMemsetAsync(c->ub.p, 0xff, comps_bound * sizeof(unsigned long long), c->stream));
    CK(cudaMemsetAsync(c->best.p, 0xff, comps_bound * sizeof(EdgeKey), c->stream));
    c->round = round;
    c->round_comps = comps_guess;   // (steers the window seeds only)
    prepare_bounds(c, n, bounds, &ms_bounds, comps_bound == n ? kLabelsNone : skip ? kLabelsFrontier : kLabelsFull);
  };
  while (comps > 1) {
    st->iterations++;
    if (st->iterations > max_it) fail(EMST_ERR_ITER, "exceeded the %d-iteration bound for n=%lld", max_it, n);
    if (!prepped) queue_bounds(st->iterations, comps, comps);
    prepped = false;
    c->round = st->iterations;
    c->round_comps = comps;
    c->one_side = comps == 2 && c->last_round_one_side;
    if (c->one_side) {
      // the component with more slots is the one left out (picked on the device: no host sync)
      CK(cudaMemsetAsync(dev_counter(c, 12), 0, sizeof(long long), c->stream));
      launch(c, k_count_label, (unsigned)c->num_sms * 4, 256, 0, (const int*)c->label.p, n, 1,
             reinterpret_cast<unsigned long long*>(dev_counter(c, 12)));
      launch(c, k_pick_side, 1, 32, 0, (const unsigned long long*)dev_counter(c, 12), n, (int*)dev_counter(c, 13));
    }
    {
      const LabelMode mode = comps == n ? kLabelsNone : skip ? kLabelsFrontier : kLabelsFull;
      exchange_bounds(c, bounds, &ms_bounds);
      prepare_labels(c, n, &ms_labels, skip && comps < n, mode);
    }
    cudaEvent_t f0 = timer_event(c);
    c->singleton_round = comps == n;
    round_find(c, n, comps, flags);
    c->one_side = false;
    c->singleton_round = false;
    c->round = 0;
    c->timers.push_back({f0, timer_event(c), &ms_find, false, st->iterations, 0, 0});
    long long emitted = 0;
    const long long bound_next = comps / 2;   // (every component merges with at least one other)
    const int it = st->iterations;
    if (bound_next > 1 && it < max_it)
      // (components shrink 3-4x per round: a quarter guesses the window-seed decision the exact
      // count would make)
      c->next_round = [&, it, bound_next] { queue_bounds(it + 1, bound_next, bound_next / 2); prepped = true; };
    long long next = round_merge(c, n, comps, edges, &emitted, &ms_merge, comps == n);
    c->next_round = nullptr;
    if (st->iterations <= 64) {
      const int r = st->iterations - 1;
      st->round_traverse_ms[r] = c->traverse_ms - tv_before;
      st->round_node_visits[r] = c->host_counters[5] - visits_before;
      st->round_found[r] = c->host_counters[6] - found_before;
      st->round_skipped[r] = c->host_counters[9] - skipped_before;
      c->skip_frac = (double)st->round_skipped[r] / (double)std::max<long long>(1, n / std::max(1, c->world));
      skipped_before = c->host_counters[9];
      visits_before = c->host_counters[5];
      found_before = c->host_counters[6];
      tv_before = c->traverse_ms;
    }
    if (c->host_counters[3]) fail(EMST_ERR_STACK, "edge traversal exceeded %d stacked nodes", kStackCapacity);
    if (next >= comps) fail(EMST_ERR_NO_REDUCE, "merge did not reduce the component count");
    edges += emitted;
    comps = next;
    if (st->num_counts < 64) st->component_counts[st->num_counts++] = comps;
  }
  if (edges != n - 1) fail(EMST_ERR_COUNT, "collected %lld edges for %lld points", edges, n);
  // packed host output: the emit and the total are left to emit_chunked, behind which the copies start
  const bool defer = packed && c->emit_overlap;
  c->emit_deferred = false;
  sort_and_emit(c, edges, edges_dev, w_dev, packed, defer);
  if (!defer) total_weight(c, w_dev, edges, st);
  CK(cudaEventRecord(t2, c->stream));
  CK(cudaEventSynchronize(t2));
  read_counters(c);
  if (sort_overflowed(c)) {   // a run of > kBlockTie equal f32 weight keys: the exact two-key order
    sort_and_emit_exact(c, edges, edges_dev, w_dev, packed);
    total_weight(c, w_dev, edges, st);
    CK(cudaEventRecord(t2, c->stream));
    CK(cudaEventSynchronize(t2));
    read_counters(c);
  } else if (defer) {
    c->emit_deferred = true;
  }
  long long evals = c->host_counters[0];
  if (c->world > 1) {
    // total work counter over ranks (instrumentation only)
    allreduce_u64(c, reinterpret_cast<unsigned long long*>(dev_counter(c, 0)), 1, 1, 0, true);
    read_counters(c);
    evals = c->host_counters[0];
  }
  st->leaf_distance_evals = evals;
  if (c->trace) {
    fprintf(stderr, "[emst] merge-to-next-round gaps: %.3f ms in all\n", c->gap_ms);
    fprintf(stderr, "[emst] final order: longest equal-key run %u, runs of 257..4096: %u, 33..256: %u, 9..32: %u\n",
            (unsigned)(c->host_counters[7] & 0xffffffffll), (unsigned)((unsigned long long)c->host_counters[7] >> 32),
            (unsigned)((unsigned long long)c->host_counters[11] >> 32), (unsigned)(c->host_counters[11] & 0xffffffffll));
  }
  c->gap_ms = 0.0;
  c->merge_end = nullptr;
#ifdef EMST_VISIT_HIST
  if (c->trace) visit_hist_print(c);
#endif
  float ms_tree = 0, ms_mst = 0;
  float ms_core = 0;
  CK(cudaEventElapsedTime(&ms_tree, t0, t3));
  CK(cudaEventElapsedTime(&ms_core, t3, t1));
  CK(cudaEventElapsedTime(&ms_mst, t1, t2));
  st->phase_ms[EMST_PHASE_TREE] = ms_tree;
  st->phase_ms[EMST_PHASE_CORE] = ms_core;
  st->phase_ms[EMST_PHASE_REDUCE_LABELS] = ms_labels;
  st->phase_ms[EMST_PHASE_UPPER_BOUNDS] = ms_bounds;
  st->phase_ms[EMST_PHASE_FIND_EDGES] = ms_find;
  st->phase_ms[EMST_PHASE_MERGE] = ms_merge;
  st->phase_ms[EMST_PHASE_MST] = ms_mst;
  st->phase_ms[EMST_PHASE_TOTAL] = ms_tree + ms_core + ms_mst;
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  cudaEventDestroy(t2);
  cudaEventDestroy(t3);
}

int finish(const Failure& f, char* err, size_t errlen) {
  if (err && errlen) snprintf(err, errlen, "%s", f.msg);
  return f.code;
}

void set_device(emst_context* c) { CK(cudaSetDevice(c->device)); }

}  // namespace

// ====================================================================== C ABI
extern "C" {

// ---- text I/O (textio.h): the reference's write_edges / write_points formats
// Formats into a library-owned buffer; *out / *len stay valid until the next
// call on any thread's behalf or emst_text_free().  (Host-only work.)
static std::string g_text;
int emst_format_edges(const int64_t* edges, const double* weights, int64_t m, const char** out, int64_t* len) {
  if (m < 0 || (m > 0 && (!edges || !weights))) return EMST_ERR_PARAM;
  g_text = emst_io::format_edges(edges, weights, m);
  *out = g_text.data();
  *len = (int64_t)g_text.size();
  return EMST_OK;
}
int emst_format_points(const float* pts, int64_t n, int32_t d, const char** out, int64_t* len) {
  if (n < 0 || (d != 2 && d != 3) || (n > 0 && !pts)) return EMST_ERR_PARAM;
  g_text = emst_io::format_points(pts, n, d);
  *out = g_text.data();
  *len = (int64_t)g_text.size();
  return EMST_OK;
}
void emst_text_free(void) { std::string().swap(g_text); }

int emst_count_rows(const char* text, int64_t len, int64_t* rows) {
  if (len < 0 || (len > 0 && !text) || !rows) return EMST_ERR_PARAM;
  *rows = emst_io::count_rows(text, text + len);
  return EMST_OK;
}

int emst_parse_rows(const char* text, int64_t len, int64_t start, int64_t line0, int64_t row0, int32_t kind,
                    int32_t width, void* out_a, void* out_b, int64_t cap, int64_t* result) {
  if (len < 0 || start < 0 || start > len || (len > 0 && !text) || !result || (kind != 0 && kind != 1)) return EMST_ERR_PARAM;
  if (kind == 1 && width != 0 && width != 2 && width != 3) return EMST_ERR_PARAM;
  if (!out_a || (kind == 0 && !out_b)) return EMST_ERR_PARAM;
  const emst_io::ParseStop st =
      emst_io::parse_csv(text, len, start, line0, row0, kind == 0, width, out_a, out_b, cap);
  if (st.line == -2) return EMST_ERR_PARAM;   // outputs too small
  result[0] = st.rows;
  result[1] = st.line;
  result[2] = st.begin;
  result[3] = st.end;
  result[4] = st.next;
  result[5] = st.width;
  return EMST_OK;
}

const char* emst_build_info(void) { return "emst_b200 sm_100a onesweep-lbvh-boruvka v1"; }

int emst_nccl_unique_id(void* id_out_128, char* err, size_t errlen) {
  try {
    ncclUniqueId id;
    NK(ncclGetUniqueId(&id));
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL id size");
    memcpy(id_out_128, &id, sizeof(id));
    return EMST_OK;
  } catch (const Failure& f) {
    return finish(f, err, errlen);
  }
}

int emst_context_create(int device, int rank, int world, const void* nccl_id, emst_context** out, char* err,
                        size_t errlen) {
  emst_context* c = nullptr;
  try {
    if (world < 1 || rank < 0 || rank >= world) fail(EMST_ERR_PARAM, "bad rank %d / world %d", rank, world);
    c = new emst_context();
    c->device = device;
    if (const char* t = getenv("EMST_SEED_WINDOW")) c->seed_window = atoi(t);
    if (const char* t = getenv("EMST_SEED_FROM")) c->seed_from = atoi(t);
    if (const char* t = getenv("EMST_SEED_WINDOW_2D")) c->seed_window_2d = atoi(t);
    if (const char* t = getenv("EMST_PROOF_FROM")) c->proof_from = atoi(t);
    if (const char* t = getenv("EMST_TRACE")) c->trace = atoi(t) != 0;
    if (const char* t = getenv("EMST_ONE_SIDE")) c->last_round_one_side = atoi(t) != 0;
    if (const char* t = getenv("EMST_IPERM_PARTS")) c->iperm_parts = atoi(t);
    if (const char* t = getenv("EMST_LIST_SKIP")) c->list_skip = atof(t);
    if (const char* t = getenv("EMST_SINGLE_KERNEL")) c->single_kernel = atoi(t) != 0;
    if (const char* t = getenv("EMST_STAGE")) c->staging = atoi(t) != 0;
    if (const char* t = getenv("EMST_EMIT_OVERLAP")) c->emit_overlap = atoi(t) != 0;
    if (const char* t = getenv("EMST_PACKED")) c->packed_out = atoi(t) != 0;
    c->rank = rank;
    c->world = world;
    set_device(c);
    CK(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    c->stream = c->own_stream;
    CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    CK(cudaMallocHost(&c->host_counters, kCounters * sizeof(long long)));
    CK(cudaEventCreate(&c->ev_a));
    CK(cudaEventCreate(&c->ev_b));
    c->counters.ensure(kCounters);
    if (world > 1 && nccl_id) {   // (without an id: a host exchange must be set, emst_context_set_exchange)
      ncclUniqueId id;
      memcpy(&id, nccl_id, sizeof(id));
      NK(ncclCommInitRank(&c->comm, world, id, rank));
    }
    *out = c;
    return EMST_OK;
  } catch (const Failure& f) {
    if (c) emst_context_destroy(c);
    return finish(f, err, errlen);
  }
}

int emst_context_destroy(emst_context* c) {
  if (!c) return EMST_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->comm) ncclCommDestroy(c->comm);
  c->pts.release(); c->scene.release(); c->part_lo.release(); c->part_hi.release(); c->part_bad.release();
  c->k0.release(); c->k1.release(); c->v0.release(); c->v1.release();
  c->sort_hist.release(); c->sort_off.release(); c->sort_status.release(); c->sort_misc.release();
  c->ident.release(); c->ident_n = 0;
  c->spts.release(); c->perm.release(); c->iperm.release(); c->nodes.release(); c->range.release();
  c->node_parent.release(); c->leaf_parent.release(); c->node_delta.release(); c->up.release(); c->arrivals.release(); c->root_box.release();
  c->label.release(); c->bprefix.release(); c->big_tops.release(); c->top.release();
  c->front[0].release(); c->front[1].release(); c->core_slot.release(); c->core_tmp.release(); c->nfn_lb.release(); c->qlist.release(); c->ub.release(); c->best.release(); c->shard_keys.release();
  c->succ.release(); c->ptr.release(); c->root.release(); c->newid.release(); c->fin.release();
  c->eout.release(); c->xw.release(); c->xuv.release(); c->exch_host.release();
  c->stager.release();
  c->scan_scratch.release(); c->counters.release(); c->out_edges.release(); c->out_w.release(); c->pairwise.release(); c->tie_runs.release(); c->tie_mid.release(); c->tie_small.release();
  if (c->host_counters) cudaFreeHost(c->host_counters);
  if (c->ev_a) cudaEventDestroy(c->ev_a);
  if (c->ev_b) cudaEventDestroy(c->ev_b);
  for (cudaEvent_t e : c->emit_ev) cudaEventDestroy(e);
  c->emit_ev.clear();
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  if (c->own_stream) cudaStreamDestroy(c->own_stream);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  delete c;
  return EMST_OK;
}

int emst_context_set_stream(emst_context* c, void* stream) {
  if (!c) return EMST_ERR_PARAM;
  c->stream = stream ? reinterpret_cast<cudaStream_t>(stream) : c->own_stream;
  return EMST_OK;
}

int emst_context_set_virtual_shards(emst_context* c, int shards) {
  if (!c || shards < 1 || shards > 64) return EMST_ERR_PARAM;
  try {
    set_device(c);
    if (shards > 1 && c->world == 1 && !c->comm) {
      // a 1-rank communicator: the virtual-shard runs take the same NCCL call path as N ranks
      int dev = c->device;
      NK(ncclCommInitAll(&c->comm, 1, &dev));
    }
  } catch (const Failure&) {
    return EMST_ERR_NCCL;
  }
  c->vshards = shards;
  return EMST_OK;
}

int emst_context_set_exchange(emst_context* c, emst_exchange_fn fn, void* user) {
  if (!c) return EMST_ERR_PARAM;
  c->exch_fn = fn;
  c->exch_user = user;
  return EMST_OK;
}

int emst_tree_token(emst_context* c, int64_t* token) {
  if (!c || !token) return EMST_ERR_PARAM;
  *token = c->tree_valid ? c->tree_token : 0;
  return EMST_OK;
}
int emst_context_reuse_tree(emst_context* c, int64_t token) {
  if (!c) return EMST_ERR_PARAM;
  c->reuse_token = token;
  return EMST_OK;
}
int emst_context_set_state_on_device(emst_context* c, int on) {
  if (!c) return EMST_ERR_PARAM;
  c->state_on_device = on != 0;
  return EMST_OK;
}

int emst_context_wait_stream(emst_context* c, void* stream) {
  if (!c) return EMST_ERR_PARAM;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (s == c->stream) return EMST_OK;
  if (cudaSetDevice(c->device) != cudaSuccess) return EMST_ERR_CUDA;
  if (cudaEventRecord(c->ev_a, s) != cudaSuccess) return EMST_ERR_CUDA;
  if (cudaStreamWaitEvent(c->stream, c->ev_a, 0) != cudaSuccess) return EMST_ERR_CUDA;
  return EMST_OK;
}

}  // extern "C"

namespace {
int boruvka_impl(emst_context* c, const float* pts, int64_t n, int32_t d, int32_t flags, int64_t k_pts,
                 const double* core_host, int64_t* edges_out, double* weights_out, emst_stats* stats, char* err,
                 size_t errlen) {
  emst_stats local;
  emst_stats* st = stats ? stats : &local;
  memset(st, 0, sizeof(*st));
  st->world = c ? c->world : 1;
  st->rank = c ? c->rank : 0;
  try {
    if (!c) fail(EMST_ERR_PARAM, "null context");
    set_device(c);
    check_shape(n, d);
    const long long launches0 = c->launches;
    c->traverse_ms = 0.0;
    c->traverse_launches = 0;
    c->traverse_queries = 0;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, c->stream));
    const float* dp = stage_points(c, pts, n, d, flags, st);
    const long long ne = n - 1;
    long long* edst;
    double* wdst;
    if (flags & EMST_OUTPUT_ON_DEVICE) {
      edst = reinterpret_cast<long long*>(edges_out);
      wdst = weights_out;
    } else {
      c->out_edges.ensure(2 * std::max<long long>(ne, 1));
      c->out_w.ensure(std::max<long long>(ne, 1));
      edst = c->out_edges.p;
      wdst = c->out_w.p;
    }
    if (n == 1) {
      // a single point has an empty tree and no iterations (mst.py:671)
      ensure_build(c, n, d);
      CK(cudaMemsetAsync(c->scene.p, 0, sizeof(Scene), c->stream));
      if (d == 3) launch(c, k_scene<3>, 1, kSceneThreads, 0, dp, n, c->part_lo.p, c->part_hi.p, c->part_bad.p, c->scene.p);
      else launch(c, k_scene<2>, 1, kSceneThreads, 0, dp, n, c->part_lo.p, c->part_hi.p, c->part_bad.p, c->scene.p);
      Scene sc;
      CK(cudaMemcpyAsync(&sc, c->scene.p, sizeof(Scene), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      if (sc.bad_row != 0x7fffffffffffffffll) fail(EMST_ERR_NONFINITE, "point %lld has a non-finite coordinate", sc.bad_row);
      st->component_counts[0] = 1;
      st->num_counts = 1;
    } else {
      const bool host_out = !(flags & EMST_OUTPUT_ON_DEVICE);
      const bool packed = host_out && c->staging && c->packed_out;
      solve(c, dp, n, d, flags, edst, wdst, st, k_pts, core_host, packed);
      c->core = nullptr;
      if (host_out) CK(cudaStreamSynchronize(c->stream));   // (host_out_ms: the transfers alone)
      const auto t_out0 = std::chrono::steady_clock::now();
      if (packed) {
        // (u << 32 | v) rows widened on the host while the next chunk is in flight (hostio.h)
        CK(c->stager.init());
        const bool w_direct = emst_host::is_pinned(weights_out);
        const bool chunked = c->emit_deferred;
        // chunked: the final emit runs chunk by chunk on the compute stream, each chunk's copy waits
        // only for its own emit (copy stream), and the total weight follows the last chunk
        const size_t per = c->stager.kSlotBytes / sizeof(unsigned long long);
        const cudaEvent_t* ready = nullptr;
        if (chunked) {
          const long long chunks = (ne + (long long)per - 1) / (long long)per;
          while ((long long)c->emit_ev.size() < chunks) {
            cudaEvent_t e;
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            c->emit_ev.push_back(e);
          }
          for (long long k = 0; k < chunks; ++k) {
            const long long i0 = k * (long long)per, i1 = std::min<long long>(ne, i0 + (long long)per);
            launch(c, k_edge_emit_packed, grid_for(i1 - i0, 256), 256, 0, c->emit_order, (const EdgeKey*)c->eout.p,
                   c->emit_key, ne, reinterpret_cast<unsigned long long*>(edst), wdst, i0, i1);
            CK(cudaEventRecord(c->emit_ev[k], c->stream));
          }
          total_weight(c, wdst, ne, st);
          ready = c->emit_ev.data();
        }
        if (w_direct) {   // page-locked destination: straight DMA, concurrent with the edge chunks below
          if (chunked) {
            CK(cudaMemcpyAsync(weights_out, wdst, ne * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
          } else {
            CK(cudaEventRecord(c->ev_b, c->stream));
            CK(cudaStreamWaitEvent(c->copy_stream, c->ev_b, 0));
            CK(cudaMemcpyAsync(weights_out, wdst, ne * sizeof(double), cudaMemcpyDeviceToHost, c->copy_stream));
          }
        }
        int64_t* eo = edges_out;
        double* wo = weights_out;
        std::vector<emst_host::Stager::Out> outs;
        outs.push_back({edst, (size_t)ne, sizeof(unsigned long long),
                        [eo](size_t at, const unsigned char* src, size_t cnt) {
                          emst_host::widen_pairs(reinterpret_cast<const unsigned long long*>(src), cnt, eo + 2 * at);
                        },
                        ready, per});
        if (!w_direct)
          outs.push_back({wdst, (size_t)ne, sizeof(double),
                          [wo](size_t at, const unsigned char* src, size_t cnt) { memcpy(wo + at, src, cnt * 8); },
                          ready, per});
        CK(c->stager.d2h(outs, chunked ? c->copy_stream : c->stream));
        if (chunked) {
          c->emit_deferred = false;
          CK(cudaStreamSynchronize(c->copy_stream));   // (c->stream is synchronised below)
        } else if (w_direct) {
          CK(cudaStreamSynchronize(c->copy_stream));
        }
        st->d2h_bytes += ne * (sizeof(unsigned long long) + sizeof(double));
      } else if (host_out) {
        CK(cudaMemcpyAsync(edges_out, edst, 2 * ne * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(weights_out, wdst, ne * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        st->d2h_bytes += ne * (2 * sizeof(long long) + sizeof(double));
      }
      if (host_out) {
        CK(cudaStreamSynchronize(c->stream));
        st->host_out_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_out0).count();
      }
    }
    CK(cudaEventRecord(e1, c->stream));
    CK(cudaEventSynchronize(e1));
    float total = 0.f;
    CK(cudaEventElapsedTime(&total, e0, e1));
    st->phase_ms[EMST_PHASE_TOTAL] = total;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    st->kernel_launches = c->launches - launches0;
    st->traverse_ms = c->traverse_ms;
    st->traverse_launches = c->traverse_launches;
    st->traverse_queries = c->traverse_queries;
    return EMST_OK;
  } catch (const Failure& f) {
    if (f.code == EMST_ERR_NONFINITE) {
      long long row = -1;
      sscanf(f.msg, "point %lld", &row);
      st->bad_row = row;
    }
    if (c) {
      c->core = nullptr;
      cudaStreamSynchronize(c->stream);
      c->timers.clear();   // (they may point at the failed solve's locals)
      c->ev_next = 0;
    }
    return finish(f, err, errlen);
  }
}
}  // namespace

extern "C" {

int emst_boruvka(emst_context* c, const float* pts, int64_t n, int32_t d, int32_t flags, int64_t* edges_out,
                 double* weights_out, emst_stats* stats, char* err, size_t errlen) {
  return boruvka_impl(c, pts, n, d, flags, 1, nullptr, edges_out, weights_out, stats, err, errlen);
}

int emst_boruvka_mrd(emst_context* c, const float* pts, int64_t n, int32_t d, int32_t flags, int64_t k_pts,
                     const double* core, int64_t* edges_out, double* weights_out, emst_stats* stats, char* err,
                     size_t errlen) {
  if (!core && k_pts < 1) {
    if (err && errlen) snprintf(err, errlen, "k_pts must be >= 1, got %lld", (long long)k_pts);
    return EMST_ERR_PARAM;
  }
  return boruvka_impl(c, pts, n, d, flags, k_pts, core, edges_out, weights_out, stats, err, errlen);
}

int emst_core_distances(emst_context* c, const float* pts, int64_t n, int32_t d, int32_t flags, int64_t k_pts,
                        double* core_out, char* err, size_t errlen) {
  try {
    if (!c) fail(EMST_ERR_PARAM, "null context");
    set_device(c);
    check_shape(n, d);
    if (k_pts < 1 || k_pts > n) fail(EMST_ERR_PARAM, "k_pts must be in [1, %lld], got %lld", (long long)n, (long long)k_pts);
    if (k_pts == 1) {   // the nearest neighbour counting self is self (metric.py:219-221)
      memset(core_out, 0, n * sizeof(double));
      return EMST_OK;
    }
    const float* dp = stage_points(c, pts, n, d, flags, nullptr);
    build_tree(c, dp, n, d);
    CK(cudaMemsetAsync(c->counters.p, 0, kCounters * sizeof(long long), c->stream));
    prepare_cores(c, n, k_pts, nullptr);
    c->core = nullptr;
    c->core_tmp.ensure(n);
    launch(c, k_scatter_by_perm, grid_for(n, 256), 256, 0, (const double*)c->core_slot.p, (const unsigned*)c->perm.p,
           n, c->core_tmp.p);
    CK(cudaMemcpyAsync(core_out, c->core_tmp.p, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return EMST_OK;
  } catch (const Failure& f) {
    if (c) {
      c->core = nullptr;
      cudaStreamSynchronize(c->stream);
      c->timers.clear();   // (they may point at the failed solve's locals)
      c->ev_next = 0;
    }
    return finish(f, err, errlen);
  }
}


}  // extern "C"

namespace {
// Morton codes of the points into c->k0: against the tight scene box (k_scene,
// which also checks finiteness), or against caller bounds (geometry.py:209-227:
// lo and 1/extent in f64, 0 on a zero-extent axis; points outside are clamped).
void codes_into_k0(emst_context* c, const float* dp, long long n, int d, const double* blo, const double* bhi) {
  ensure_build(c, n, d);
  CK(cudaMemsetAsync(c->scene.p, 0, sizeof(Scene), c->stream));
  unsigned sg = (unsigned)std::min<long long>(grid_for(n, kSceneThreads), (long long)c->num_sms * 8);
  if (d == 3) launch(c, k_scene<3>, sg, kSceneThreads, 0, dp, n, c->part_lo.p, c->part_hi.p, c->part_bad.p, c->scene.p);
  else launch(c, k_scene<2>, sg, kSceneThreads, 0, dp, n, c->part_lo.p, c->part_hi.p, c->part_bad.p, c->scene.p);
  Scene sc;
  CK(cudaMemcpyAsync(&sc, c->scene.p, sizeof(Scene), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (sc.bad_row != 0x7fffffffffffffffll) fail(EMST_ERR_NONFINITE, "point %lld has a non-finite coordinate", sc.bad_row);
  if (blo) {
    for (int k = 0; k < 3; ++k) {
      const double lo = k < d ? blo[k] : 0.0, hi = k < d ? bhi[k] : 0.0;
      if (!(lo <= hi)) fail(EMST_ERR_PARAM, "bounds have lo > hi on axis %d", k);
      const double ext = hi - lo;
      sc.lo[k] = lo;
      sc.inv[k] = ext > 0.0 ? 1.0 / ext : 0.0;
    }
    CK(cudaMemcpyAsync(c->scene.p, &sc, sizeof(Scene), cudaMemcpyHostToDevice, c->stream));
  }
  if (d == 3) launch(c, k_morton<3>, grid_for(n, 256), 256, 0, dp, n, (const Scene*)c->scene.p, c->k0.p);
  else launch(c, k_morton<2>, grid_for(n, 256), 256, 0, dp, n, (const Scene*)c->scene.p, c->k0.p);
}
}  // namespace

extern "C" {

int emst_morton_codes(emst_context* c, const float* pts, int64_t n, int32_t d, int32_t flags, const double* bounds_lo,
                      const double* bounds_hi, uint64_t* codes_out, char* err, size_t errlen) {
  try {
    if (!c) fail(EMST_ERR_PARAM, "null context");
    set_device(c);
    check_shape(n, d);
    if (!bounds_lo != !bounds_hi) fail(EMST_ERR_PARAM, "give both bound corners or neither");
    const float* dp = stage_points(c, pts, n, d, flags, nullptr);
    codes_into_k0(c, dp, n, d, bounds_lo, bounds_hi);
    CK(cudaMemcpyAsync(codes_out, c->k0.p, n * sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return EMST_OK;
  } catch (const Failure& f) {
    if (c) cudaStreamSynchronize(c->stream);
    return finish(f, err, errlen);
  }
}

int emst_sort_by_morton(emst_context* c, const float* pts, int64_t n, int32_t d, int32_t flags, const double* bounds_lo,
                        const double* bounds_hi, int64_t* perm_out, char* err, size_t errlen) {
  try {
    if (!c) fail(EMST_ERR_PARAM, "null context");
    set_device(c);
    check_shape(n, d);
    if (!bounds_lo != !bounds_hi) fail(EMST_ERR_PARAM, "give both bound corners or neither");
    const float* dp = stage_points(c, pts, n, d, flags, nullptr);
    codes_into_k0(c, dp, n, d, bounds_lo, bounds_hi);
    unsigned long long* keys;
    unsigned* order;
    radix_sort(c, n, d == 3 ? 63 : 62, c->k0.p, c->v0.p, true, c->k1.p, c->v1.p, &keys, &order);
    DevBuf<long long> wide;
    wide.ensure(n);
    launch(c, k_u32_to_i64, grid_for(n, 256), 256, 0, (const unsigned*)order, (long long)n, wide.p);
    CK(cudaMemcpyAsync(perm_out, wide.p, n * sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    wide.release();
    return EMST_OK;
  } catch (const Failure& f) {
    if (c) cudaStreamSynchronize(c->stream);
    return finish(f, err, errlen);
  }
}

int emst_build(emst_context* c, const float* pts, int64_t n, int32_t d, int32_t flags, int64_t* perm, int64_t* left,
               int64_t* right, int64_t* parent, int64_t* leaf_parent, float* box_lo, float* box_hi,
               int64_t* sweep_order, int64_t* sweep_starts, int64_t* n_starts, char* err, size_t errlen) {
  try {
    if (!c) fail(EMST_ERR_PARAM, "null context");
    set_device(c);
    check_shape(n, d);
    const float* dp = stage_points(c, pts, n, d, flags, nullptr);
    build_tree(c, dp, n, d);
    const long long m = n - 1;
    // export in the reference's int64 layout through scratch device buffers
    DevBuf<long long> tmp;
    tmp.ensure((size_t)(4 * std::max<long long>(m, 1) + n));
    DevBuf<float> boxes;
    boxes.ensure((size_t)2 * std::max<long long>(m, 1) * d);
    long long *dl = tmp.p, *dr = dl + std::max<long long>(m, 1), *dpar = dr + std::max<long long>(m, 1),
              *dlp = dpar + std::max<long long>(m, 1);
    if (d == 3)
      launch(c, k_export_tree<Node3>, grid_for(n, 256), 256, 0, (const Node3*)reinterpret_cast<Node3*>(c->nodes.p),
             (const int*)c->node_parent.p, (const int*)c->leaf_parent.p, n, (const Box3*)c->root_box.p, dl, dr, dpar,
             dlp, boxes.p, boxes.p + std::max<long long>(m, 1) * d, d);
    else
      launch(c, k_export_tree<Node2>, grid_for(n, 256), 256, 0, (const Node2*)reinterpret_cast<Node2*>(c->nodes.p),
             (const int*)c->node_parent.p, (const int*)c->leaf_parent.p, n, (const Box3*)c->root_box.p, dl, dr, dpar,
             dlp, boxes.p, boxes.p + std::max<long long>(m, 1) * d, d);
    std::vector<unsigned> hperm(n);
    CK(cudaMemcpyAsync(hperm.data(), c->perm.p, n * sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream));
    if (m > 0) {
      CK(cudaMemcpyAsync(left, dl, m * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaMemcpyAsync(right, dr, m * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaMemcpyAsync(parent, dpar, m * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaMemcpyAsync(box_lo, boxes.p, m * d * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaMemcpyAsync(box_hi, boxes.p + std::max<long long>(m, 1) * d, m * d * sizeof(float),
                         cudaMemcpyDeviceToHost, c->stream));
    }
    CK(cudaMemcpyAsync(leaf_parent, dlp, n * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (long long i = 0; i < n; ++i) perm[i] = hperm[i];
    if (n == 1) leaf_parent[0] = -1;
    if (sweep_order && sweep_starts && n_starts) {
      // the level schedule: heights by arrival climb, stable sort of the heights (bvh.py:204-238, 293-302)
      *n_starts = 1;
      sweep_starts[0] = 0;
      if (m > 0) {
        DevBuf<unsigned> height;
        height.ensure(m);
        CK(cudaMemsetAsync(height.p, 0, m * sizeof(unsigned), c->stream));
        CK(cudaMemsetAsync(c->arrivals.p, 0, m * sizeof(unsigned), c->stream));
        launch(c, k_node_heights, grid_for(n, 256), 256, 0, (const int*)c->leaf_parent.p, (const int*)c->node_parent.p,
               (long long)n, c->arrivals.p, height.p);
        launch(c, k_u32_to_u64, grid_for(m, 256), 256, 0, (const unsigned*)height.p, m, c->k0.p);
        unsigned long long* hs;
        unsigned* order;
        radix_sort(c, m, 32, c->k0.p, c->v0.p, true, c->k1.p, c->v1.p, &hs, &order);
        DevBuf<long long> out;
        out.ensure(2 * m + 1);
        launch(c, k_level_starts, grid_for(m, 256), 256, 0, (const unsigned long long*)hs, (const unsigned*)order, m,
               out.p + m, out.p);
        unsigned long long hmax = 0;
        CK(cudaMemcpyAsync(&hmax, hs + (m - 1), sizeof(hmax), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(sweep_order, out.p, m * sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (hmax < 1 || hmax > (unsigned long long)m) fail(EMST_ERR_COUNT, "node height %llu out of range", hmax);
        CK(cudaMemcpyAsync(sweep_starts, out.p + m, (hmax + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        *n_starts = (int64_t)hmax + 1;
        height.release();
        out.release();
      }
    }
    tmp.release();
    boxes.release();
    return EMST_OK;
  } catch (const Failure& f) {
    if (c) cudaStreamSynchronize(c->stream);
    return finish(f, err, errlen);
  }
}

}  // extern "C"

// ---------------------------------------------- per-round building blocks
// These operate on reference-layout state: labels are representative point
// indices (any value < n works as an identifier), per-component arrays are
// n-sized and indexed by label.  Slot-space labels are gathered through perm.

namespace {

// coarsening check of the kept proofs: a previous label l names a point of its component (the
// reference's labels are member indices); every slot must share its new label with the slot of
// that point, iperm[l] (any violation, of either kind, -> *flag: the proofs are dropped)
__global__ void k_bb_check(const int* __restrict__ prev, const int* __restrict__ label,
                           const unsigned* __restrict__ iperm, long long n, int* __restrict__ flag) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= n) return;
  const int l = prev[s];
  const unsigned r = iperm[l];
  if (prev[r] != l || label[r] != label[s]) *flag = 1;
}
// every point its own component (labels are the points' own indices): *flag = 1 otherwise
__global__ void k_bb_singletons(const int* __restrict__ label, const unsigned* __restrict__ perm, long long n,
                                int* __restrict__ flag) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s < n && label[s] != (int)perm[s]) *flag = 1;
}

template <class Node>
__global__ void k_reset_node_labels(Node* __restrict__ nodes, long long m) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < m) *reinterpret_cast<int2*>(&nodes[i].ref.z) = make_int2(kMixed, kMixed);
}

__global__ void k_labels_to_slots(const long long* __restrict__ labels_pt, const unsigned* __restrict__ perm, long long n,
                                  int* __restrict__ label_slot) {
  long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s < n) label_slot[s] = (int)labels_pt[perm[s]];
}

template <class Node>
__global__ void k_export_node_labels(const Node* __restrict__ nodes, long long m, const long long* __restrict__ labels_pt,
                                     const unsigned* __restrict__ perm, const int* __restrict__ node_parent,
                                     const int* __restrict__ label_slot, const int2* __restrict__ range,
                                     const int* __restrict__ bprefix, long long* __restrict__ il) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= m) return;
  // node i's own label is held in its parent's record; the root's is derived directly
  if (i == 0) {
    int2 r = range[0];
    il[0] = bprefix[r.y] == bprefix[r.x] ? (long long)label_slot[r.x] : (long long)kMixed;
    return;
  }
  int link = node_parent[i];
  int4 ref = nodes[link >> 1].ref;
  il[i] = (link & 1) ? ref.w : ref.z;
}

void prepare_labels_from_host(emst_context* c, const int64_t* labels, long long n) {
  ensure_rounds(c, n);
  CK(cudaMemsetAsync(c->nfn_lb.p, 0, n * sizeof(float), c->stream));
  if (c->state_on_device) {   // caller's device array: no staging
    launch(c, k_labels_to_slots, grid_for(n, 256), 256, 0, (const long long*)labels, (const unsigned*)c->perm.p, n,
           c->label.p);
    return;
  }
  DevBuf<long long> lab;
  lab.ensure(n);
  CK(cudaMemcpyAsync(lab.p, labels, n * sizeof(long long), cudaMemcpyHostToDevice, c->stream));
  launch(c, k_labels_to_slots, grid_for(n, 256), 256, 0, (const long long*)lab.p, (const unsigned*)c->perm.p, n, c->label.p);
  CK(cudaStreamSynchronize(c->stream));
  lab.release();
}

// The tree a building block works on: the context's current one when the
// caller named it (emst_context_reuse_tree, one call), else built from pts.
void tree_for_call(emst_context* c, const float* pts, long long n, int d) {
  const bool reuse = c->reuse_token != 0 && c->reuse_token == c->tree_token && c->tree_valid && c->n == n &&
                     c->dim == d;
  c->reuse_token = 0;
  if (reuse) return;
  const float* dp = stage_points(c, pts, n, d, 0, nullptr);
  build_tree(c, dp, n, d);
}

// f64 bound bits of the device state -> the traversal's u64 radii (inf / NaN / negative: none)
__global__ void k_bounds_in(const double* __restrict__ ub, long long n, bool use, unsigned long long* __restrict__ bits) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double w = use ? ub[i] : __longlong_as_double(0x7ff0000000000000ll);
  bits[i] = (w >= 0.0 && w < __longlong_as_double(0x7ff0000000000000ll)) ? (unsigned long long)__double_as_longlong(w) : ~0ull;
}
__global__ void k_bounds_out(const unsigned long long* __restrict__ bits, long long n, double* __restrict__ ub) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long b = bits[i] >= 0x7ff0000000000000ull ? 0x7ff0000000000000ull : bits[i];
  ub[i] = __longlong_as_double((long long)b);
}
__global__ void k_best_out(const EdgeKey* __restrict__ best, long long n, long long* __restrict__ bu,
                           long long* __restrict__ bv, double* __restrict__ bw) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const EdgeKey k = best[i];
  const bool none = k.uv == ~0ull;
  bu[i] = none ? -1 : (long long)(k.uv >> 32);
  bv[i] = none ? -1 : (long long)(k.uv & 0xffffffffull);
  bw[i] = none ? __longlong_as_double(0x7ff0000000000000ll) : __longlong_as_double((long long)k.w);
}

}  // namespace

extern "C" {

int emst_reduce_labels(emst_context* c, const float* pts, int64_t n, int32_t d, const int64_t* labels,
                       int64_t* internal_labels, char* err, size_t errlen) {
  try {
    set_device(c);
    check_shape(n, d);
    tree_for_call(c, pts, n, d);
    if (n == 1) return EMST_OK;
    prepare_labels_from_host(c, labels, n);
    round_prepare(c, n, false, nullptr, nullptr);
    DevBuf<long long> il;
    long long* ild = reinterpret_cast<long long*>(internal_labels);
    if (!c->state_on_device) {
      il.ensure(n - 1);
      ild = il.p;
    }
    if (d == 3)
      launch(c, k_export_node_labels<Node3>, grid_for(n - 1, 256), 256, 0, (const Node3*)reinterpret_cast<Node3*>(c->nodes.p),
             n - 1, (const long long*)nullptr, (const unsigned*)c->perm.p, (const int*)c->node_parent.p,
             (const int*)c->label.p, (const int2*)c->range.p, (const int*)c->bprefix.p, ild);
    else
      launch(c, k_export_node_labels<Node2>, grid_for(n - 1, 256), 256, 0, (const Node2*)reinterpret_cast<Node2*>(c->nodes.p),
             n - 1, (const long long*)nullptr, (const unsigned*)c->perm.p, (const int*)c->node_parent.p,
             (const int*)c->label.p, (const int2*)c->range.p, (const int*)c->bprefix.p, ild);
    if (!c->state_on_device)
      CK(cudaMemcpyAsync(internal_labels, il.p, (n - 1) * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    il.release();
    return EMST_OK;
  } catch (const Failure& f) {
    if (c) cudaStreamSynchronize(c->stream);
    return finish(f, err, errlen);
  }
}

int emst_compute_upper_bounds(emst_context* c, const float* pts, int64_t n, int32_t d, const int64_t* labels,
                              const double* core, double* ub_out, char* err, size_t errlen) {
  try {
    set_device(c);
    check_shape(n, d);
    tree_for_call(c, pts, n, d);
    prepare_labels_from_host(c, labels, n);
    CK(cudaMemsetAsync(c->ub.p, 0xff, n * sizeof(unsigned long long), c->stream));
    prepare_cores(c, n, 1, core);
    round_prepare(c, n, true, nullptr, nullptr);
    c->core = nullptr;
    if (c->state_on_device) {
      launch(c, k_bounds_out, grid_for(n, 256), 256, 0, (const unsigned long long*)c->ub.p, n, ub_out);
      CK(cudaStreamSynchronize(c->stream));
      return EMST_OK;
    }
    std::vector<unsigned long long> bits(n);
    CK(cudaMemcpyAsync(bits.data(), c->ub.p, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (long long i = 0; i < n; ++i) {
      unsigned long long b = bits[i] >= 0x7ff0000000000000ull ? 0x7ff0000000000000ull : bits[i];
      memcpy(&ub_out[i], &b, 8);
    }
    return EMST_OK;
  } catch (const Failure& f) {
    if (c) cudaStreamSynchronize(c->stream);
    return finish(f, err, errlen);
  }
}

int emst_find_component_outgoing_edges(emst_context* c, const float* pts, int64_t n, int32_t d, const int64_t* labels,
                                       const double* ub, const double* core, int32_t flags, int64_t* best_u,
                                       int64_t* best_v, double* best_w, int64_t* leaf_evals, char* err,
                                       size_t errlen) {
  try {
    set_device(c);
    check_shape(n, d);
    if (n < 2) fail(EMST_ERR_NOTHING, "a single component has no outgoing edges");
    tree_for_call(c, pts, n, d);
    prepare_labels_from_host(c, labels, n);
    if (c->state_on_device) {
      launch(c, k_bounds_in, grid_for(n, 256), 256, 0, ub, n, (flags & EMST_UPPER_BOUNDS) != 0, c->ub.p);
    } else {
      std::vector<unsigned long long> bits(n);
      for (long long i = 0; i < n; ++i) {
        double w = (flags & EMST_UPPER_BOUNDS) ? ub[i] : __builtin_inf();
        memcpy(&bits[i], &w, 8);
        if (!(w >= 0.0) || w == __builtin_inf()) bits[i] = ~0ull;
      }
      CK(cudaMemcpyAsync(c->ub.p, bits.data(), n * sizeof(unsigned long long), cudaMemcpyHostToDevice, c->stream));
      CK(cudaStreamSynchronize(c->stream));   // (bits is a local)
    }
    // node labels only (bounds are caller-provided).  With subtree_skip the labelling is
    // the solve's frontier form over every node (pure subtrees become "inside", top pure
    // nodes are recorded, so queries whose search box stays inside theirs settle at once);
    // it starts from MIXED records, as after a build
    const bool skip = flags & EMST_SUBTREE_SKIP;
    if (skip && n > 1) {
      if (d == 3) launch(c, k_reset_node_labels<Node3>, grid_for(n - 1, 256), 256, 0, reinterpret_cast<Node3*>(c->nodes.p), n - 1);
      else launch(c, k_reset_node_labels<Node2>, grid_for(n - 1, 256), 256, 0, reinterpret_cast<Node2*>(c->nodes.p), n - 1);
      CK(cudaMemsetAsync(c->top.p, 0, n * sizeof(int), c->stream));
      c->front_n = -1;
    }
    round_prepare(c, n, false, nullptr, nullptr, skip, skip ? kLabelsFrontier : kLabelsFull);
    CK(cudaMemsetAsync(c->best.p, 0xff, n * sizeof(EdgeKey), c->stream));
    CK(cudaMemsetAsync(c->counters.p, 0, kCounters * sizeof(long long), c->stream));
    prepare_cores(c, n, 1, core);
    c->one_side = false;
    // nearest-foreign proofs (Euclidean, single rank): kept from the previous call on this tree
    // when its components are coarsened by these, else started afresh
    const bool proofs = (flags & EMST_UPPER_BOUNDS) && !core && c->world == 1 && c->vshards == 1 && c->proof_from > 0;
    if (proofs) {
      c->bb_nfn.ensure(n);
      c->bb_prev.ensure(n);
      bool keep = c->bb_token == c->tree_token;
      if (keep) {
        int* flag = reinterpret_cast<int*>(dev_counter(c, 15));
        launch(c, k_bb_check, grid_for(n, 256), 256, 0, (const int*)c->bb_prev.p, (const int*)c->label.p,
               (const unsigned*)c->iperm.p, (long long)n, flag);
        read_counters(c);
        keep = c->host_counters[15] == 0;
        CK(cudaMemsetAsync(flag, 0, sizeof(long long), c->stream));
      }
      if (!keep) {
        CK(cudaMemsetAsync(c->bb_nfn.p, 0, n * sizeof(float), c->stream));
        c->bb_skip = 0.0;
        c->bb_calls = 0;
        // a chain starts: all singletons is the solve's round 1 (its own kernel)
        int* flag = reinterpret_cast<int*>(dev_counter(c, 15));
        launch(c, k_bb_singletons, grid_for(n, 256), 256, 0, (const int*)c->label.p, (const unsigned*)c->perm.p,
               (long long)n, flag);
        read_counters(c);
        c->singleton_round = c->host_counters[15] == 0;
        CK(cudaMemsetAsync(flag, 0, sizeof(long long), c->stream));
      }
      std::swap(c->nfn_lb, c->bb_nfn);
      // the chain's k-th call runs as the solve's round k: the proof kernel from proof_from on,
      // query lists once the previous call settled enough queries up front
      c->round = c->bb_calls + 1;
      c->skip_frac = c->bb_skip;
    }
    round_find(c, n, n, flags);
    c->singleton_round = false;
    if (proofs) {
      std::swap(c->nfn_lb, c->bb_nfn);
      c->round = 0;
      c->bb_calls++;
      CK(cudaMemcpyAsync(c->bb_prev.p, c->label.p, n * sizeof(int), cudaMemcpyDeviceToDevice, c->stream));
      c->bb_token = c->tree_token;
    }
    c->core = nullptr;
    if (c->state_on_device) {
      launch(c, k_best_out, grid_for(n, 256), 256, 0, (const EdgeKey*)c->best.p, n, reinterpret_cast<long long*>(best_u),
             reinterpret_cast<long long*>(best_v), best_w);
      read_counters(c);
      if (c->host_counters[3]) fail(EMST_ERR_STACK, "edge traversal exceeded %d stacked nodes", kStackCapacity);
      if (leaf_evals) *leaf_evals = c->host_counters[0];
      if (proofs) c->bb_skip = (double)c->host_counters[9] / (double)n;
      return EMST_OK;
    }
    std::vector<EdgeKey> keys(n);
    CK(cudaMemcpyAsync(keys.data(), c->best.p, n * sizeof(EdgeKey), cudaMemcpyDeviceToHost, c->stream));
    read_counters(c);
    if (c->host_counters[3]) fail(EMST_ERR_STACK, "edge traversal exceeded %d stacked nodes", kStackCapacity);
    if (proofs) c->bb_skip = (double)c->host_counters[9] / (double)n;
    for (long long i = 0; i < n; ++i) {
      if (keys[i].uv == ~0ull) {
        best_u[i] = -1;
        best_v[i] = -1;
        best_w[i] = __builtin_inf();
      } else {
        best_u[i] = (long long)(keys[i].uv >> 32);
        best_v[i] = (long long)(keys[i].uv & 0xffffffffull);
        memcpy(&best_w[i], &keys[i].w, 8);
      }
    }
    if (leaf_evals) *leaf_evals = c->host_counters[0];
    return EMST_OK;
  } catch (const Failure& f) {
    if (c) {
      c->bb_token = 0;   // (the proof buffers may be swapped)
      c->round = 0;
      c->singleton_round = false;
    }
    if (c) cudaStreamSynchronize(c->stream);
    return finish(f, err, errlen);
  }
}

}  // extern "C"

namespace {
__global__ void k_cluster_min(const int* __restrict__ ptr, const long long* __restrict__ reps, long long s,
                              long long* __restrict__ cmin) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k < s) atomicMin(&cmin[ptr[k]], reps[k]);
}

// ---- merge_components on device state (all arrays device-resident)
// dense[reps[k]] = k; err bit 1: a representative out of range, bit 2: listed twice
__global__ void k_dense_map(const long long* __restrict__ reps, long long s, long long n, int* __restrict__ dense,
                            int* __restrict__ err) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= s) return;
  const long long r = reps[k];
  if (r < 0 || r >= n) { atomicOr(err, 1); return; }
  if (atomicExch(&dense[r], (int)k) != -1) atomicOr(err, 2);
}
// label[i] = dense[labels[i]]; err bit 4: a label that is not a listed representative
__global__ void k_dense_labels(const long long* __restrict__ labels, long long n, const int* __restrict__ dense,
                               int* __restrict__ label, int* __restrict__ err) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long l = labels[i];
  const int k = (l >= 0 && l < n) ? dense[l] : -1;
  if (k < 0) atomicOr(err, 4);
  label[i] = k < 0 ? 0 : k;
}
// per dense component: its best edge as a 128-bit key; err bit 8: an endpoint out of range
__global__ void k_keys_from_best(const long long* __restrict__ reps, long long s, const long long* __restrict__ bu,
                                 const long long* __restrict__ bv, const double* __restrict__ bw, long long n,
                                 EdgeKey* __restrict__ best, int* __restrict__ err) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= s) return;
  const long long r = reps[k];
  EdgeKey e;
  e.uv = ~0ull;
  e.w = ~0ull;
  if (r >= 0 && r < n && bv[r] >= 0) {
    const long long u = bu[r], v = bv[r];
    if (u < 0 || u >= n || v >= n) atomicOr(err, 8);
    else {
      e.uv = ((unsigned long long)u << 32) | (unsigned long long)v;
      e.w = (unsigned long long)__double_as_longlong(bw[r]);
    }
  }
  best[k] = e;
}
// reference labels: every point adopts its cluster's smallest representative
// (the dense slot labels were already relabelled by the merge: go through the input labels again)
__global__ void k_labels_from_clusters(long long* __restrict__ labels, long long n, const int* __restrict__ dense,
                                       const int* __restrict__ root, const long long* __restrict__ cmin) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) labels[i] = cmin[root[dense[labels[i]]]];
}
__global__ void k_edges_out(const EdgeKey* __restrict__ eout, long long ne, long long* __restrict__ ou,
                            long long* __restrict__ ov, double* __restrict__ ow) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= ne) return;
  const EdgeKey k = eout[e];
  ou[e] = (long long)(k.uv >> 32);
  ov[e] = (long long)(k.uv & 0xffffffffull);
  ow[e] = __longlong_as_double((long long)k.w);
}
// new_reps: the representatives that are their cluster's minimum, in k (= ascending) order
struct NewRepsOp {
  using T = unsigned;
  static constexpr bool kCached = false;
  static constexpr bool kWarpStore = false;
  const int* root;
  const long long* reps;
  const long long* cmin;
  long long* new_reps;
  long long s;
  __device__ void load(long long i0, int cnt, unsigned* v) const {
#pragma unroll
    for (int j = 0; j < kScanItems; ++j)
      v[j] = j < cnt && cmin[root[i0 + j]] == reps[i0 + j] ? 1u : 0u;
  }
  __device__ void side(long long, int, const unsigned*) const {}
  __device__ void store(long long i0, int cnt, const unsigned* v, unsigned ex) const {
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
      if (j < cnt && v[j]) new_reps[ex] = reps[i0 + j];
      ex += v[j];
    }
  }
};

// identity permutation of n (point order is the merge building block's "slot" order; the
// tree's own iperm stays intact for the calls that reuse the tree)
const unsigned* identity_perm(emst_context* c, long long n) {
  if (c->ident_n < n) {
    c->ident.ensure(n);
    launch(c, k_iota_u32, grid_for(n, 256), 256, 0, c->ident.p, n);
    c->ident_n = n;
  }
  return c->ident.p;
}

void merge_on_device(emst_context* c, long long n, const long long* reps, long long s, const long long* bu,
                     const long long* bv, const double* bw, long long* labels, long long* out_u, long long* out_v,
                     double* out_w, long long* n_edges, long long* new_reps, long long* n_new) {
  int* dense = c->bprefix.p;   // (n ints; the merge does not use the boundary prefix)
  int* err = reinterpret_cast<int*>(dev_counter(c, 2)) + 1;   // high word of counters[2]
  CK(cudaMemsetAsync(c->counters.p, 0, kCounters * sizeof(long long), c->stream));
  CK(cudaMemsetAsync(dense, 0xff, n * sizeof(int), c->stream));
  launch(c, k_dense_map, grid_for(s, 256), 256, 0, reps, s, n, dense, err);
  launch(c, k_dense_labels, grid_for(n, 256), 256, 0, (const long long*)labels, n, (const int*)dense, c->label.p, err);
  launch(c, k_keys_from_best, grid_for(s, 256), 256, 0, reps, s, bu, bv, bw, n, c->best.p, err);
  read_counters(c);
  const int e = (int)((unsigned long long)c->host_counters[2] >> 32);
  if (e & 1) fail(EMST_ERR_PARAM, "a representative is out of range [0, %lld)", n);
  if (e & 2) fail(EMST_ERR_PARAM, "a representative is listed twice");
  if (e & 4) fail(EMST_ERR_PARAM, "a label is not a listed representative");
  if (e & 8) fail(EMST_ERR_PARAM, "a component's edge has an endpoint out of range");
  long long emitted = 0;
  const long long next = round_merge(c, n, s, 0, &emitted, nullptr, false, identity_perm(c, n));
  if (next >= s) fail(EMST_ERR_NO_REDUCE, "merge did not reduce the component count");
  long long* cmin = reinterpret_cast<long long*>(c->ub.p);   // (s words; the merge does not use the bounds)
  CK(cudaMemsetAsync(cmin, 0x7f, s * sizeof(long long), c->stream));
  launch(c, k_cluster_min, grid_for(s, 256), 256, 0, (const int*)c->root.p, reps, s, cmin);
  launch(c, k_labels_from_clusters, grid_for(n, 256), 256, 0, labels, n, (const int*)dense, (const int*)c->root.p,
         (const long long*)cmin);
  run_scan(c, s, NewRepsOp{c->root.p, reps, cmin, new_reps, s}, false);
  if (emitted) launch(c, k_edges_out, grid_for(emitted, 256), 256, 0, (const EdgeKey*)c->eout.p, emitted, out_u, out_v, out_w);
  CK(cudaStreamSynchronize(c->stream));
  *n_edges = emitted;
  *n_new = next;
}
}  // namespace

extern "C" int emst_merge_components(emst_context* c, int64_t n, const int64_t* reps, int64_t s, const int64_t* best_u,
                                     const int64_t* best_v, const double* best_w, int64_t* labels, int64_t* out_u,
                                     int64_t* out_v, double* out_w, int64_t* n_edges, int64_t* new_reps,
                                     int64_t* n_new, char* err, size_t errlen) {
  // Dense-id formulation of mst.py:517-547: component k <-> reps[k].
  try {
    set_device(c);
    if (s < 1 || n < 1) fail(EMST_ERR_PARAM, "empty merge");
    ensure_rounds(c, n);
    c->counters.ensure(kCounters);
    if (s > n) fail(EMST_ERR_PARAM, "%lld representatives for %lld points", (long long)s, (long long)n);
    if (c->state_on_device) {
      long long ne = 0, nn = 0;
      merge_on_device(c, n, reinterpret_cast<const long long*>(reps), s, reinterpret_cast<const long long*>(best_u),
                      reinterpret_cast<const long long*>(best_v), best_w, reinterpret_cast<long long*>(labels),
                      reinterpret_cast<long long*>(out_u), reinterpret_cast<long long*>(out_v), out_w, &ne,
                      reinterpret_cast<long long*>(new_reps), &nn);
      *n_edges = ne;
      *n_new = nn;
      return EMST_OK;
    }
    std::vector<int> dense(n, -1), lab(n);
    for (long long k = 0; k < s; ++k) {
      const long long r = reps[k];
      if (r < 0 || r >= n) fail(EMST_ERR_PARAM, "representative %lld out of range [0, %lld)", r, (long long)n);
      if (dense[r] >= 0) fail(EMST_ERR_PARAM, "representative %lld listed twice", r);
      dense[r] = (int)k;
    }
    for (long long i = 0; i < n; ++i) {
      const long long l = labels[i];
      if (l < 0 || l >= n || dense[l] < 0)
        fail(EMST_ERR_PARAM, "label %lld of point %lld is not a listed representative", l, i);
      lab[i] = dense[l];
    }
    std::vector<EdgeKey> keys(s);
    for (long long k = 0; k < s; ++k) {
      long long r = reps[k];
      if (best_v[r] < 0) { keys[k].uv = ~0ull; keys[k].w = ~0ull; continue; }
      if (best_u[r] < 0 || best_u[r] >= n || best_v[r] >= n)
        fail(EMST_ERR_PARAM, "edge (%lld, %lld) of component %lld out of range", (long long)best_u[r],
             (long long)best_v[r], r);
      keys[k].uv = ((unsigned long long)best_u[r] << 32) | (unsigned long long)best_v[r];
      memcpy(&keys[k].w, &best_w[r], 8);
    }
    CK(cudaMemcpyAsync(c->label.p, lab.data(), n * sizeof(int), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->best.p, keys.data(), s * sizeof(EdgeKey), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemsetAsync(c->counters.p, 0, kCounters * sizeof(long long), c->stream));
    long long emitted = 0;
    long long next = round_merge(c, n, s, 0, &emitted, nullptr, false, identity_perm(c, n));
    if (next >= s) fail(EMST_ERR_NO_REDUCE, "merge did not reduce the component count");
    // reference labels: each cluster adopts its smallest representative
    DevBuf<long long> dreps, cmin;
    dreps.ensure(s);
    cmin.ensure(s);
    CK(cudaMemcpyAsync(dreps.p, reps, s * sizeof(long long), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemsetAsync(cmin.p, 0x7f, s * sizeof(long long), c->stream));
    launch(c, k_cluster_min, grid_for(s, 256), 256, 0, (const int*)c->root.p, (const long long*)dreps.p, s, cmin.p);
    std::vector<int> ptr(s), newlab(n);
    std::vector<long long> cm(s);
    std::vector<EdgeKey> eo(emitted);
    CK(cudaMemcpyAsync(ptr.data(), c->root.p, s * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(cm.data(), cmin.p, s * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
    if (emitted) {
      CK(cudaMemcpyAsync(eo.data(), c->eout.p, emitted * sizeof(EdgeKey), cudaMemcpyDeviceToHost, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    for (long long i = 0; i < n; ++i) {
      int k = lab[i];
      labels[i] = k >= 0 ? cm[ptr[k]] : labels[i];
    }
    long long nn = 0;
    for (long long k = 0; k < s; ++k)
      if (ptr[k] == (int)k) new_reps[nn++] = cm[k];
    std::sort(new_reps, new_reps + nn);
    for (long long e = 0; e < emitted; ++e) {
      out_u[e] = (long long)(eo[e].uv >> 32);
      out_v[e] = (long long)(eo[e].uv & 0xffffffffull);
      memcpy(&out_w[e], &eo[e].w, 8);
    }
    *n_edges = emitted;
    *n_new = nn;
    dreps.release();
    cmin.release();
    return EMST_OK;
  } catch (const Failure& f) {
    if (c) cudaStreamSynchronize(c->stream);
    return finish(f, err, errlen);
  }
}
