/*
 * emst_b200.h -- C ABI of the B200-native single-tree Boruvka EMST.
 *
 * Plain pointers and sizes only (no torch / numpy types).  Each entry point
 * replaces one function of the reference package (/root/reference/pkg/src/emst);
 * the citation next to it is the reference interface it stands in for.  The
 * Python drop-in (paper_2207_00514_b200/) binds these with ctypes, see
 * INTEGRATION.md.
 *
 * Conventions
 *   - points are row-major float32 (n, d), d in {2, 3}; every output array is
 *     caller-allocated with the documented size.
 *   - EMST_POINTS_ON_DEVICE: `pts` is a CUDA device pointer (zero-copy hand-off
 *     of a contiguous float32 CUDA tensor); otherwise a host pointer.
 *   - EMST_OUTPUT_ON_DEVICE: edges/weights outputs are device pointers.
 *   - every call returns an emst_status; on failure `err` (if non-NULL) holds a
 *     NUL-terminated message.  No call falls back to the CPU.
 *   - a context is bound to one CUDA device and one stream; calls on one context
 *     must be serialised by the caller (the Python layer holds a lock).
 */
#ifndef EMST_B200_H
#define EMST_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum emst_status {
  EMST_OK = 0,
  EMST_ERR_EMPTY = 1,          /* EmptyDatasetError          (geometry.py:64-65)   */
  EMST_ERR_DIM = 2,            /* UnsupportedDimensionError  (geometry.py:59-67)   */
  EMST_ERR_NONFINITE = 3,      /* InvalidCoordinateError     (geometry.py:68-70)   */
  EMST_ERR_STACK = 4,          /* TraversalStackOverflowError (mst.py:705-707)     */
  EMST_ERR_NO_EDGE = 5,        /* InternalInvariantViolation (mst.py:720-721)      */
  EMST_ERR_CHAIN = 6,          /* InternalInvariantViolation (mst.py:722-723)      */
  EMST_ERR_NO_REDUCE = 7,      /* InternalInvariantViolation (mst.py:724-725)      */
  EMST_ERR_ITER = 8,           /* InternalInvariantViolation (mst.py:682-684)      */
  EMST_ERR_COUNT = 9,          /* InternalInvariantViolation (mst.py:742-744)      */
  EMST_ERR_CUDA = 10,          /* DeviceError (new)                                */
  EMST_ERR_NCCL = 11,          /* DeviceError (new)                                */
  EMST_ERR_PARAM = 12,         /* InvalidParameterError                            */
  EMST_ERR_TOO_LARGE = 13,     /* InvalidParameterError: n beyond 2^30 - 1         */
  EMST_ERR_NOTHING = 14,       /* NothingToFindError         (mst.py:487-488)      */
  EMST_ERR_MISSING = 15        /* NoOutgoingEdgeError        (mst.py:510-513)      */
} emst_status;

enum {
  EMST_SUBTREE_SKIP = 1,        /* boruvka_emst(subtree_skip=True)        mst.py:579 */
  EMST_UPPER_BOUNDS = 2,        /* boruvka_emst(upper_bound_seeding=True) mst.py:580 */
  EMST_POINTS_ON_DEVICE = 4,
  EMST_OUTPUT_ON_DEVICE = 8
};

/* Phase slots of emst_stats.phase_ms, the keys of MstResult.phase_timings (mst.py:756-765). */
enum {
  EMST_PHASE_TREE = 0, EMST_PHASE_CORE = 1, EMST_PHASE_REDUCE_LABELS = 2, EMST_PHASE_UPPER_BOUNDS = 3,
  EMST_PHASE_FIND_EDGES = 4, EMST_PHASE_MERGE = 5, EMST_PHASE_MST = 6, EMST_PHASE_TOTAL = 7
};

/* Run instrumentation, the non-array fields of MstResult (mst.py:158-182). */
typedef struct emst_stats {
  int32_t iterations;
  int32_t num_counts;
  int64_t component_counts[64];
  int64_t leaf_distance_evals;
  double phase_ms[8];
  int64_t bad_row;              /* first non-finite row when EMST_ERR_NONFINITE */
  int64_t kernel_launches;      /* kernels this call launched */
  int64_t h2d_bytes;
  int64_t d2h_bytes;
  int32_t world;                /* GPUs that shared the traversal */
  int32_t rank;
  double traverse_ms;           /* device time of the traversal kernel launches */
  int64_t traverse_launches;
  int64_t traverse_queries;     /* queries those launches processed (this rank) */
  double round_traverse_ms[64]; /* per Boruvka round: traversal device time */
  int64_t round_node_visits[64];/* per round: node records fetched by the traversal */
  int64_t round_found[64];      /* per round: queries that found a candidate edge */
  int64_t round_skipped[64];    /* per round: queries settled before any node visit */
  double total_weight;          /* float(np.sum(weights)): numpy's pairwise order, on the device */
  double host_in_ms;            /* host wall time handing the points over (host-pointer entry) */
  double host_out_ms;           /* host wall time bringing the edges / weights back */
} emst_stats;

typedef struct emst_context emst_context;

/* NCCL rendezvous id (128 bytes) for a multi-GPU context; rank 0 creates it and
 * the caller broadcasts it (torch.distributed in the Python layer). */
int emst_nccl_unique_id(void* id_out_128, char* err, size_t errlen);

/* One context per (process, device).  world > 1 shares every Boruvka round's
 * traversal by Morton slot range over `world` ranks (replicated tree, one
 * two-phase min-reduction per round over NCCL); nccl_id may be NULL when
 * world == 1, or when a host exchange is set (emst_context_set_exchange). */
int emst_context_create(int device, int rank, int world, const void* nccl_id, emst_context** out,
                        char* err, size_t errlen);
int emst_context_destroy(emst_context* ctx);

/* Run this context's work on an external CUDA stream (cudaStream_t; NULL restores
 * the context's own stream) -- lets a caller time calls with its own events. */
int emst_context_set_stream(emst_context* ctx, void* stream);

/* Shards per rank: each rank's part of a round's traversal is split into `shards`
 * Morton ranges (S = world * shards in all) whose per-component keys go through
 * the same two-phase exchange kernels and all-reduce as N ranks do: the local
 * rows are folded on the device, then ncclAllReduce runs on the communicator
 * (a 1-rank communicator is created for world == 1, so one GPU exercises the
 * whole N-rank path).  Determinism tests of the multi-GPU protocol use it. */
int emst_context_set_virtual_shards(emst_context* ctx, int shards);

/* Host exchange for ranks without an NCCL communicator (a context created with
 * world > 1 and nccl_id == NULL): `fn` all-reduces `count` u64 in place in
 * page-locked host memory over every rank, by unsigned min (EMST_EXCHANGE_MIN)
 * or sum (EMST_EXCHANGE_SUM), and returns 0 on success.  The Python layer binds
 * it to torch.distributed.all_reduce of any backend (gloo); it replaces
 * ncclAllReduce in the two-phase exchange of mst.py:236-348's sharded query loop. */
enum { EMST_EXCHANGE_MIN = 0, EMST_EXCHANGE_SUM = 1 };
typedef int (*emst_exchange_fn)(uint64_t* buf, int64_t count, int32_t op, void* user);
int emst_context_set_exchange(emst_context* ctx, emst_exchange_fn fn, void* user);

/* Make the context's stream wait for the work queued so far on `stream` (a
 * cudaStream_t, e.g. torch's current stream) -- call it before handing the
 * library device memory that another stream produced. */
int emst_context_wait_stream(emst_context* ctx, void* stream);

/* boruvka_emst(points, "euclidean", 1, subtree_skip, upper_bound_seeding)
 * (mst.py:578-769).  edges_out: (n-1) x 2 int64, u < v; weights_out: (n-1)
 * float64; rows sorted by (weight, u, v).  stats may be NULL. */
int emst_boruvka(emst_context* ctx, const float* pts, int64_t n, int32_t d, int32_t flags,
                 int64_t* edges_out, double* weights_out, emst_stats* stats, char* err, size_t errlen);

/* boruvka_emst(points, "mrd", k_pts) or boruvka_emst(points, MutualReachability(core)) (mst.py:578-769,
 * metric.py:128-234): edge weights max(d, core(u), core(v)).  core: NULL to compute the k_pts-th nearest
 * neighbour distances (self included; 1 <= k_pts <= n, k_pts = 1 is plain Euclidean), or n f64 in
 * original point order (host).  Outputs as emst_boruvka; stats->phase_ms[EMST_PHASE_CORE] times the cores. */
int emst_boruvka_mrd(emst_context* ctx, const float* pts, int64_t n, int32_t d, int32_t flags, int64_t k_pts,
                     const double* core, int64_t* edges_out, double* weights_out, emst_stats* stats, char* err,
                     size_t errlen);

/* Text formats of the reference's writers (data.py:117-141, 222-235), formatted on all host threads:
 * emst_format_edges -> "u,v,%.17g\n" per edge; emst_format_points -> "%.9g" coordinates joined by ','
 * and '\n' per row.  *out (length *len, not NUL-terminated) is owned by the library and valid until the
 * next emst_format_* call or emst_text_free(); calls are not thread-safe. */
int emst_format_edges(const int64_t* edges, const double* weights, int64_t m, const char** out, int64_t* len);
int emst_format_points(const float* pts, int64_t n, int32_t d, const char** out, int64_t* len);
void emst_text_free(void);

/* The reference's CSV readers (data.py:148-198 read_points, 225-257 read_edges) on all host threads.
 * emst_count_rows: lines of text[0, len) that are not blank (an upper bound of the rows).
 * emst_parse_rows: parses text[start, len) -- its first line numbered line0 -- into rows [row0, cap):
 * kind 0 edges "u,v,w" (out_a int64 (m, 2), out_b f64 (m)), kind 1 points (out_a f32 (n, width);
 * width 0 = take 2 or 3 from the first non-blank line).  Plain ASCII spellings are converted here; the
 * first line that is anything else (an error, or a spelling only Python's int()/float() take) stops the
 * parse and is handed back for the caller to apply the reference's rules to it and resume after it.
 * result[6] = {rows written in all, that line's number (-1: none), its begin, end (terminator
 * excluded), the offset to resume at, the row width}. */
int emst_count_rows(const char* text, int64_t len, int64_t* rows);
int emst_parse_rows(const char* text, int64_t len, int64_t start, int64_t line0, int64_t row0, int32_t kind,
                    int32_t width, void* out_a, void* out_b, int64_t cap, int64_t* result);

/* compute_core_distances(build(points), points, k_pts) (metric.py:209-234): core_out n f64 (host), original
 * point order; k_pts in [1, n] (EMST_ERR_PARAM otherwise). */
int emst_core_distances(emst_context* ctx, const float* pts, int64_t n, int32_t d, int32_t flags, int64_t k_pts,
                        double* core_out, char* err, size_t errlen);

/* morton_codes(points, bounds) (geometry.py:209-227). codes_out: n u64 (host).  bounds_lo / bounds_hi:
 * d f64 each (an Aabb; points outside are clamped into it), or both NULL for the tight scene box. */
int emst_morton_codes(emst_context* ctx, const float* pts, int64_t n, int32_t d, int32_t flags,
                      const double* bounds_lo, const double* bounds_hi, uint64_t* codes_out, char* err,
                      size_t errlen);

/* sort_by_morton(points, bounds) (geometry.py:247-254): the stable (code, index) order, perm_out n int64
 * (host); bounds as emst_morton_codes.  The GPU onesweep sort of the solve. */
int emst_sort_by_morton(emst_context* ctx, const float* pts, int64_t n, int32_t d, int32_t flags,
                        const double* bounds_lo, const double* bounds_hi, int64_t* perm_out, char* err,
                        size_t errlen);

/* build(points) (bvh.py:305-340) in the reference's array layout (bvh.py:39-75):
 * perm n, left/right/parent n-1, leaf_parent n (int64); box_lo/box_hi (n-1) x d f32. Host outputs.
 * sweep_order (n-1) and sweep_starts (capacity n) receive the level schedule (bvh.py:293-302),
 * *n_starts its length (height + 1); pass three NULLs to skip it. */
int emst_build(emst_context* ctx, const float* pts, int64_t n, int32_t d, int32_t flags, int64_t* perm,
               int64_t* left, int64_t* right, int64_t* parent, int64_t* leaf_parent, float* box_lo,
               float* box_hi, int64_t* sweep_order, int64_t* sweep_starts, int64_t* n_starts, char* err,
               size_t errlen);

/* reduce_labels(build(points), state) (mst.py:436-448): labels n int64 (point order) -> internal labels n-1. */
int emst_reduce_labels(emst_context* ctx, const float* pts, int64_t n, int32_t d, const int64_t* labels,
                       int64_t* internal_labels, char* err, size_t errlen);

/* compute_upper_bounds(state, build(points).leaf_perm, points) (mst.py:451-469): ub_out n f64 by label. */
int emst_compute_upper_bounds(emst_context* ctx, const float* pts, int64_t n, int32_t d, const int64_t* labels,
                              const double* core, double* ub_out, char* err, size_t errlen);

/* find_component_outgoing_edges (mst.py:472-514): per-label best edge arrays (n each, -1 / inf
 * where none), flags as emst_boruvka; ub is read only with EMST_UPPER_BOUNDS.  core (both functions):
 * NULL for Euclidean, else n f64 core distances in point order (mutual reachability). */
int emst_find_component_outgoing_edges(emst_context* ctx, const float* pts, int64_t n, int32_t d,
                                       const int64_t* labels, const double* ub, const double* core, int32_t flags,
                                       int64_t* best_u, int64_t* best_v, double* best_w, int64_t* leaf_evals,
                                       char* err, size_t errlen);

/* merge_components (mst.py:517-547): reps (s, ascending), per-label best arrays (n); labels
 * (n) relabelled in place; out_u/out_v/out_w (s) and new_reps (s) with their counts. */
int emst_merge_components(emst_context* ctx, int64_t n, const int64_t* reps, int64_t s, const int64_t* best_u,
                          const int64_t* best_v, const double* best_w, int64_t* labels, int64_t* out_u,
                          int64_t* out_v, double* out_w, int64_t* n_edges, int64_t* new_reps, int64_t* n_new,
                          char* err, size_t errlen);

/* Device-resident building blocks (mst.py:436-547 called round by round without host copies):
 *  - emst_tree_token: names the tree the context holds (0: none); it changes with every build
 *    (emst_build, a solve, or a building block that had to build);
 *  - emst_context_reuse_tree: the next building-block call on this context skips its own
 *    build when `token` still names the context's tree (same points, n and d: the caller's
 *    promise, as the reference's Bvh is a snapshot of its points) -- one call only;
 *  - emst_context_set_state_on_device: while on, the state arrays the four building blocks
 *    take and return (labels, internal labels, bounds, best edges, reps, merged edges, new reps)
 *    are device pointers on the context's device; the points stay host (or the reused tree). */
int emst_tree_token(emst_context* ctx, int64_t* token);
int emst_context_reuse_tree(emst_context* ctx, int64_t token);
int emst_context_set_state_on_device(emst_context* ctx, int on);

/* Library identification: compiled arch string (e.g. "sm_100a") and a build tag. */
const char* emst_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* EMST_B200_H */
