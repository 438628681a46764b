/*
 * emst_oracle.c -- CPU restatement of the reference single-tree Boruvka EMST.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product in paper_2207_00514_b200/.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load it, and only as the
 * checker or the reported CPU baseline -- never as the thing measured or shipped.
 *
 * It restates, in plain C, the algorithm of the reference package
 * /root/reference/pkg/src/emst (numba JIT kernels), function by function; every
 * function below cites the reference file:line it follows.  The arithmetic
 * convention is the reference's: float32 coordinates, every distance evaluated
 * in float64 with a fixed per-axis summation order and no fused multiply-add
 * (compile with -ffp-contract=off, never -ffast-math; geometry.py:1-8,108-124).
 *
 * Parity is pinned in tests/test_oracle_golden.py against golden vectors that
 * tests/golden/make_goldens.py recorded by running the reference itself.
 *
 * Parallelism mirrors the reference: the loops the reference runs with numba
 * prange (Morton codes, per-level label reduction, per-query traversal, relabel)
 * are OpenMP-parallel; the loops it runs serially (upper-bound fold, candidate
 * fold, merge) stay serial, so results do not depend on the thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_MIXED (-1)        /* mst.py:57 */
#define OR_STACK 64          /* bvh.py:36 STACK_CAPACITY */

enum {
    OR_OK = 0,
    OR_ERR_STACK = 1,        /* TraversalStackOverflowError (mst.py:705-707) */
    OR_ERR_NO_EDGE = 2,      /* merge code -1 (mst.py:720-721) */
    OR_ERR_CHAIN = 3,        /* merge code -2 (mst.py:722-723) */
    OR_ERR_NO_REDUCE = 4,    /* mst.py:724-725 */
    OR_ERR_ITER = 5,         /* mst.py:682-684 */
    OR_ERR_COUNT = 6,        /* mst.py:742-744 */
    OR_ERR_ALLOC = 7,
    OR_ERR_TOPOLOGY = 8      /* bvh.py:333-337 */
};

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}

/* ------------------------------------------------------------------ Morton */

/* Tight f32 bounds widened to f64 (geometry.py:102-105). */
static void scene_bounds(const float *pts, int64_t n, int d, double *lo, double *hi) {
    for (int k = 0; k < d; ++k) {
        float mn = pts[k], mx = pts[k];
        for (int64_t i = 1; i < n; ++i) {
            float x = pts[i * d + k];
            if (x < mn) mn = x;
            if (x > mx) mx = x;
        }
        lo[k] = (double)mn;
        hi[k] = (double)mx;
    }
}

/* 1/extent, 0 on zero-extent axes (geometry.py:201-206). */
static void axis_inverses(const double *lo, const double *hi, int d, double *inv) {
    for (int k = 0; k < d; ++k) {
        double ext = hi[k] - lo[k];
        inv[k] = ext > 0.0 ? 1.0 / ext : 0.0;
    }
}

/* Quantize one coordinate to its lattice cell (geometry.py:169-177). */
static uint64_t cell_of(double x, double lo, double inv, double scale) {
    static const double below_one = 0.99999999999999988898; /* nextafter(1, 0), geometry.py:33 */
    double t = (x - lo) * inv;
    if (t < 0.0) t = 0.0;
    else if (t > below_one) t = below_one;
    return (uint64_t)(t * scale);
}

/* Axis a's bit j goes to bit j*d + (d-1-a): x most significant in each group
 * (geometry.py:143-198; the bit map is the one test_geometry.py:121-131 states). */
static uint64_t interleave(const uint64_t *cells, int d, int bits) {
    uint64_t code = 0;
    for (int a = 0; a < d; ++a)
        for (int j = 0; j < bits; ++j)
            if ((cells[a] >> j) & 1u) code |= (uint64_t)1 << (j * d + (d - 1 - a));
    return code;
}

/* morton_codes with the default (tight scene) bounds (geometry.py:209-227). */
void oracle_morton_codes(const float *pts, int64_t n, int d, uint64_t *out) {
    double lo[3], hi[3], inv[3];
    scene_bounds(pts, n, d, lo, hi);
    axis_inverses(lo, hi, d, inv);
    const int bits = d == 2 ? 31 : 21;                 /* geometry.py:28-29 */
    const double scale = (double)((uint64_t)1 << bits);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        uint64_t c[3];
        for (int k = 0; k < d; ++k) c[k] = cell_of((double)pts[i * d + k], lo[k], inv[k], scale);
        out[i] = interleave(c, d, bits);
    }
}

/* ------------------------------------------------------------ stable sorts */

/* One stable counting-sort pass on a 16-bit digit of key[idx[i]]. */
static void radix_pass(const uint64_t *key, const int64_t *src, int64_t *dst, int64_t n, int shift) {
    int64_t *cnt = (int64_t *)calloc(65537, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) cnt[((key[src[i]] >> shift) & 0xFFFF) + 1]++;
    for (int b = 0; b < 65536; ++b) cnt[b + 1] += cnt[b];
    for (int64_t i = 0; i < n; ++i) dst[cnt[(key[src[i]] >> shift) & 0xFFFF]++] = src[i];
    free(cnt);
}

/* Stable argsort on u64 keys: equals np.argsort(kind="stable") (bvh.py:317,
 * geometry.py:247-254): ties keep ascending original index. */
static int stable_argsort_u64(const uint64_t *key, int64_t n, int64_t *perm, int nbits) {
    int64_t *tmp = (int64_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    if (!tmp) return OR_ERR_ALLOC;
    for (int64_t i = 0; i < n; ++i) perm[i] = i;
    int64_t *a = perm, *b = tmp;
    int passes = 0;
    for (int shift = 0; shift < nbits; shift += 16, ++passes) {
        radix_pass(key, a, b, n, shift);
        int64_t *t = a; a = b; b = t;
    }
    if (a != perm) memcpy(perm, a, (size_t)n * sizeof(int64_t));
    free(tmp);
    return OR_OK;
}

void oracle_sort_by_morton(const float *pts, int64_t n, int d, int64_t *perm) {
    uint64_t *codes = (uint64_t *)malloc((size_t)n * sizeof(uint64_t));
    oracle_morton_codes(pts, n, d, codes);
    stable_argsort_u64(codes, n, perm, 64);
    free(codes);
}

/* --------------------------------------------------------------- topology */

/* Common-prefix length of the augmented keys (code, position) at sorted
 * positions i and j, -1 out of range (bvh.py:112-149). */
static inline int prefix_len(const uint64_t *codes, int64_t n, int64_t i, int64_t j) {
    if (j < 0 || j >= n) return -1;
    uint64_t a = codes[i], b = codes[j];
    if (a != b) return __builtin_clzll(a ^ b);
    return 64 + __builtin_clzll((uint64_t)i ^ (uint64_t)j);
}

/* Karras radix-tree topology of sorted codes (bvh.py:152-201).  Packed refs:
 * < m internal, >= m leaf slot + m; root is internal node 0. */
static void karras_topology(const uint64_t *sc, int64_t n, int64_t *left, int64_t *right,
                            int64_t *parent, int64_t *leaf_parent) {
    const int64_t m = n - 1;
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i) {
        int dir = prefix_len(sc, n, i, i + 1) > prefix_len(sc, n, i, i - 1) ? 1 : -1;
        int floor_len = prefix_len(sc, n, i, i - dir);
        /* grow an upper bound on the range length, then bisect for its end */
        int64_t span = 2;
        while (prefix_len(sc, n, i, i + span * dir) > floor_len) span <<= 1;
        int64_t len = 0;
        for (int64_t step = span >> 1; step >= 1; step >>= 1)
            if (prefix_len(sc, n, i, i + (len + step) * dir) > floor_len) len += step;
        int64_t j = i + len * dir;
        /* bisect for the split: furthest position still sharing more than the node prefix */
        int node_len = prefix_len(sc, n, i, j);
        int64_t s = 0, step = len;
        while (step > 1) {
            step = (step + 1) >> 1;
            if (prefix_len(sc, n, i, i + (s + step) * dir) > node_len) s += step;
        }
        int64_t gamma = i + s * dir + (dir < 0 ? -1 : 0);
        int64_t lo = i < j ? i : j, hi = i < j ? j : i;
        if (lo == gamma) { left[i] = m + gamma; leaf_parent[gamma] = i; }
        else { left[i] = gamma; parent[gamma] = i; }
        if (hi == gamma + 1) { right[i] = m + gamma + 1; leaf_parent[gamma + 1] = i; }
        else { right[i] = gamma + 1; parent[gamma + 1] = i; }
    }
}

/* Height levels: nodes of height h depend only on lower levels
 * (bvh.py:204-238, 293-302).  Returns the number of resolved nodes. */
static int64_t level_schedule(const int64_t *left, const int64_t *right, const int64_t *parent,
                              int64_t m, int64_t *order, int64_t *starts, int *nlevels) {
    int64_t *h = (int64_t *)calloc((size_t)m, sizeof(int64_t));
    int64_t *ready = (int64_t *)calloc((size_t)m, sizeof(int64_t));
    int64_t *queue = (int64_t *)malloc((size_t)m * sizeof(int64_t));
    int64_t tail = 0, head = 0;
    for (int64_t v = 0; v < m; ++v) {
        ready[v] = (left[v] >= m) + (right[v] >= m);
        if (ready[v] == 2) { h[v] = 1; queue[tail++] = v; }
    }
    while (head < tail) {
        int64_t v = queue[head++];
        int64_t p = parent[v];
        if (p < 0) continue;
        if (++ready[p] == 2) {
            int64_t hl = left[p] >= m ? 0 : h[left[p]];
            int64_t hr = right[p] >= m ? 0 : h[right[p]];
            h[p] = 1 + (hl > hr ? hl : hr);
            queue[tail++] = p;
        }
    }
    int64_t hmax = 0;
    for (int64_t v = 0; v < m; ++v) if (h[v] > hmax) hmax = h[v];
    /* counting sort of nodes by height (stable, like np.argsort(kind="stable")) */
    int64_t *cnt = (int64_t *)calloc((size_t)hmax + 2, sizeof(int64_t));
    for (int64_t v = 0; v < m; ++v) cnt[h[v]]++;
    int64_t acc = 0;
    for (int64_t k = 0; k <= hmax; ++k) { int64_t c = cnt[k]; cnt[k] = acc; acc += c; }
    for (int64_t k = 1; k <= hmax; ++k) starts[k - 1] = cnt[k];
    starts[hmax] = m;
    for (int64_t v = 0; v < m; ++v) order[cnt[h[v]]++] = v;
    *nlevels = (int)hmax;
    free(cnt); free(h); free(ready); free(queue);
    return tail;
}

typedef struct {
    int64_t n, m;
    int d;
    int64_t *perm, *left, *right, *parent, *leaf_parent;
    float *box_lo, *box_hi;
    int64_t *order, *starts;
    int nlevels;
} or_tree;

/* Bottom-up f32 min/max per level (bvh.py:241-264). */
static void refit(or_tree *t, const float *pts) {
    const int64_t m = t->m;
    const int d = t->d;
    for (int lev = 0; lev < t->nlevels; ++lev) {
        #pragma omp parallel for schedule(static)
        for (int64_t oi = t->starts[lev]; oi < t->starts[lev + 1]; ++oi) {
            int64_t v = t->order[oi];
            int64_t c[2] = {t->left[v], t->right[v]};
            for (int k = 0; k < d; ++k) {
                float lo[2], hi[2];
                for (int s = 0; s < 2; ++s) {
                    if (c[s] >= m) lo[s] = hi[s] = pts[t->perm[c[s] - m] * d + k];
                    else { lo[s] = t->box_lo[c[s] * d + k]; hi[s] = t->box_hi[c[s] * d + k]; }
                }
                t->box_lo[v * d + k] = lo[0] < lo[1] ? lo[0] : lo[1];
                t->box_hi[v * d + k] = hi[0] > hi[1] ? hi[0] : hi[1];
            }
        }
    }
}

static void tree_free(or_tree *t) {
    free(t->perm); free(t->left); free(t->right); free(t->parent); free(t->leaf_parent);
    free(t->box_lo); free(t->box_hi); free(t->order); free(t->starts);
}

/* build (bvh.py:305-340). */
static int tree_build(or_tree *t, const float *pts, int64_t n, int d) {
    memset(t, 0, sizeof(*t));
    t->n = n; t->m = n - 1; t->d = d;
    int64_t m = n - 1, mm = m > 0 ? m : 1;
    t->perm = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    t->left = (int64_t *)malloc((size_t)mm * sizeof(int64_t));
    t->right = (int64_t *)malloc((size_t)mm * sizeof(int64_t));
    t->parent = (int64_t *)malloc((size_t)mm * sizeof(int64_t));
    t->leaf_parent = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    t->box_lo = (float *)malloc((size_t)mm * d * sizeof(float));
    t->box_hi = (float *)malloc((size_t)mm * d * sizeof(float));
    t->order = (int64_t *)malloc((size_t)mm * sizeof(int64_t));
    t->starts = (int64_t *)malloc((size_t)(mm + 2) * sizeof(int64_t));
    uint64_t *codes = (uint64_t *)malloc((size_t)n * sizeof(uint64_t));
    uint64_t *sc = (uint64_t *)malloc((size_t)n * sizeof(uint64_t));
    if (!t->perm || !t->left || !t->right || !t->parent || !t->leaf_parent || !t->box_lo ||
        !t->box_hi || !t->order || !t->starts || !codes || !sc) {
        free(codes); free(sc); tree_free(t); return OR_ERR_ALLOC;
    }
    oracle_morton_codes(pts, n, d, codes);
    stable_argsort_u64(codes, n, t->perm, 64);
    for (int64_t i = 0; i < m; ++i) t->parent[i] = -1;
    for (int64_t i = 0; i < n; ++i) t->leaf_parent[i] = -1;
    t->starts[0] = 0;
    t->nlevels = 0;
    if (n > 1) {
        for (int64_t i = 0; i < n; ++i) sc[i] = codes[t->perm[i]];
        karras_topology(sc, n, t->left, t->right, t->parent, t->leaf_parent);
        int64_t roots = 0;
        for (int64_t i = 0; i < m; ++i) roots += t->parent[i] == -1;
        if (roots != 1 || t->parent[0] != -1) { free(codes); free(sc); tree_free(t); return OR_ERR_TOPOLOGY; }
        int64_t done = level_schedule(t->left, t->right, t->parent, m, t->order, t->starts, &t->nlevels);
        if (done != m) { free(codes); free(sc); tree_free(t); return OR_ERR_TOPOLOGY; }
        refit(t, pts);
    }
    free(codes); free(sc);
    return OR_OK;
}

/* Exported build: reference-layout arrays (bvh.py:39-75). */
int oracle_build(const float *pts, int64_t n, int d, int64_t *perm, int64_t *left, int64_t *right,
                 int64_t *parent, int64_t *leaf_parent, float *box_lo, float *box_hi) {
    or_tree t;
    int rc = tree_build(&t, pts, n, d);
    if (rc) return rc;
    memcpy(perm, t.perm, (size_t)n * sizeof(int64_t));
    memcpy(leaf_parent, t.leaf_parent, (size_t)n * sizeof(int64_t));
    if (n > 1) {
        memcpy(left, t.left, (size_t)(n - 1) * sizeof(int64_t));
        memcpy(right, t.right, (size_t)(n - 1) * sizeof(int64_t));
        memcpy(parent, t.parent, (size_t)(n - 1) * sizeof(int64_t));
        memcpy(box_lo, t.box_lo, (size_t)(n - 1) * d * sizeof(float));
        memcpy(box_hi, t.box_hi, (size_t)(n - 1) * d * sizeof(float));
    }
    tree_free(&t);
    return OR_OK;
}

/* ------------------------------------------------------------ round phases */

/* internal label = common child label or MIXED, children first (mst.py:185-195). */
static void reduce_labels(const or_tree *t, const int64_t *labels, int64_t *il) {
    const int64_t m = t->m;
    for (int lev = 0; lev < t->nlevels; ++lev) {
        #pragma omp parallel for schedule(static)
        for (int64_t oi = t->starts[lev]; oi < t->starts[lev + 1]; ++oi) {
            int64_t v = t->order[oi];
            int64_t lc = t->left[v], rc = t->right[v];
            int64_t ll = lc >= m ? labels[t->perm[lc - m]] : il[lc];
            int64_t rl = rc >= m ? labels[t->perm[rc - m]] : il[rc];
            il[v] = ll == rl ? ll : OR_MIXED;
        }
    }
}

/* Euclidean distance in f64, axis order, no FMA (bvh.py:284-290, geometry.py:108-124). */
static inline double point_dist(const float *pts, int d, int64_t p, const double *q) {
    double s = 0.0;
    for (int k = 0; k < d; ++k) {
        double dx = q[k] - (double)pts[p * d + k];
        s += dx * dx;
    }
    return sqrt(s);
}

/* Lower bound from q to a node's box, f64 (bvh.py:267-281). */
static inline double box_dist(const float *lo, const float *hi, int d, int64_t node, const double *q) {
    double s = 0.0;
    for (int k = 0; k < d; ++k) {
        double x = q[k], l = (double)lo[node * d + k], h = (double)hi[node * d + k];
        double dx = 0.0;
        if (x < l) dx = l - x;
        else if (x > h) dx = x - h;
        s += dx * dx;
    }
    return sqrt(s);
}

/* Adjacent Z-order pairs in different components seed both radii; serial fold
 * in slot order (mst.py:198-224).  Caller resets ub at live reps. */
static void upper_bounds(const float *pts, int d, const int64_t *perm, int64_t n, const int64_t *labels,
                         const double *cores, double *ub) {
    for (int64_t s = 0; s + 1 < n; ++s) {
        int64_t a = perm[s], b = perm[s + 1];
        int64_t la = labels[a], lb = labels[b];
        if (la == lb) continue;
        double acc = 0.0;
        for (int k = 0; k < d; ++k) {
            double dx = (double)pts[a * d + k] - (double)pts[b * d + k];
            acc += dx * dx;
        }
        double w = sqrt(acc);
        if (cores) { if (cores[a] > w) w = cores[a]; if (cores[b] > w) w = cores[b]; }
        if (w < ub[la]) ub[la] = w;
        if (w < ub[lb]) ub[lb] = w;
    }
}

/* (w, u, v) lexicographic "less than" (mst.py:62-89, 283-285). */
static inline int edge_less(double w, int64_t u, int64_t v, double bw, int64_t bu, int64_t bv) {
    return w < bw || (w == bw && (u < bu || (u == bu && v < bv)));
}

/* Per-query constrained nearest-foreign-neighbour search, Algorithm 2
 * (mst.py:227-328).  Returns the number of leaf distance evaluations;
 * sets *overflow on stack overflow. */
static int64_t find_edges(const or_tree *t, const float *pts, const int64_t *labels, const int64_t *il,
                          const double *ub, const double *cores, int use_bounds, int skip,
                          int64_t q_begin, int64_t q_end,
                          int64_t *cand_u, int64_t *cand_v, double *cand_w, int *overflow) {
    const int64_t m = t->m;
    const int d = t->d;
    int64_t evals_total = 0;
    int ovf = 0;
    #pragma omp parallel for schedule(dynamic, 4096) reduction(+ : evals_total) reduction(| : ovf)
    for (int64_t s = q_begin; s < q_end; ++s) {
        int64_t node_stack[OR_STACK];
        double dist_stack[OR_STACK];
        double q[3];
        int64_t qp = t->perm[s];
        int64_t comp = labels[qp];
        double cq = cores ? cores[qp] : 0.0;
        for (int k = 0; k < d; ++k) q[k] = (double)pts[qp * d + k];
        double radius = use_bounds ? ub[comp] : INFINITY;
        double best_w = INFINITY;
        int64_t best_u = -1, best_v = -1;
        double root_lb = box_dist(t->box_lo, t->box_hi, d, 0, q);
        if (cq > root_lb) root_lb = cq;
        node_stack[0] = 0;
        dist_stack[0] = root_lb;
        int top = 1;
        while (top > 0) {
            --top;
            if (dist_stack[top] > radius) continue;
            int64_t ref = node_stack[top];
            int64_t child[2] = {t->left[ref], t->right[ref]};
            int64_t pa = -1, pb = -1;
            double pa_d = 0.0, pb_d = 0.0;
            for (int side = 0; side < 2; ++side) {
                int64_t c = child[side];
                if (c >= m) {
                    int64_t p = t->perm[c - m];
                    double w = point_dist(pts, d, p, q);
                    evals_total++;
                    if (labels[p] == comp) continue;
                    if (cores) { if (cores[p] > w) w = cores[p]; if (cq > w) w = cq; }
                    if (w <= radius) {
                        int64_t u = qp < p ? qp : p, v = qp < p ? p : qp;
                        if (edge_less(w, u, v, best_w, best_u, best_v)) {
                            best_w = w; best_u = u; best_v = v; radius = w;
                        }
                    }
                } else {
                    if (skip && il[c] == comp) continue;
                    double bd = box_dist(t->box_lo, t->box_hi, d, c, q);
                    if (cq > bd) bd = cq;
                    if (bd <= radius) {
                        if (pa < 0) { pa = c; pa_d = bd; }
                        else { pb = c; pb_d = bd; }
                    }
                }
            }
            if (pb >= 0) {
                if (top + 2 > OR_STACK) { ovf = 1; top = 0; continue; }
                if (pb_d < pa_d) {   /* nearer child on top; ties keep the left one there */
                    int64_t tn = pa; pa = pb; pb = tn;
                    double td = pa_d; pa_d = pb_d; pb_d = td;
                }
                node_stack[top] = pb; dist_stack[top] = pb_d; ++top;
                node_stack[top] = pa; dist_stack[top] = pa_d; ++top;
            } else if (pa >= 0) {
                if (top + 1 > OR_STACK) { ovf = 1; top = 0; continue; }
                node_stack[top] = pa; dist_stack[top] = pa_d; ++top;
            }
        }
        cand_u[qp] = best_u;
        cand_v[qp] = best_v;
        cand_w[qp] = best_w;
    }
    *overflow |= ovf;
    return evals_total;
}

/* Per-component minimum under (w, u, v), serial in point order (mst.py:331-348). */
static void reduce_candidates(const int64_t *labels, int64_t n, const int64_t *cu, const int64_t *cv,
                              const double *cw, int64_t *bu, int64_t *bv, double *bw) {
    for (int64_t q = 0; q < n; ++q) {
        int64_t v = cv[q];
        if (v < 0) continue;
        int64_t c = labels[q];
        if (edge_less(cw[q], cu[q], v, bw[c], bu[c], bv[c])) { bw[c] = cw[q]; bu[c] = cu[q]; bv[c] = v; }
    }
}

/* Component-graph collapse (mst.py:351-427).  Returns edges emitted (>= 0) or
 * -1 (broken candidate) / -2 (unterminated chain); *n_new gets the survivors. */
static int64_t merge(const int64_t *reps, int64_t s, const int64_t *bu, const int64_t *bv, const double *bw,
                     const int64_t *labels, int64_t *succ, int64_t *terminal, int64_t *cluster_min,
                     int64_t *final_, int64_t *out_u, int64_t *out_v, double *out_w, int64_t *new_reps,
                     int64_t *n_new) {
    for (int64_t i = 0; i < s; ++i) {
        int64_t r = reps[i];
        terminal[r] = -1;
        cluster_min[r] = -1;
        if (bv[r] < 0) return -1;
        int64_t lu = labels[bu[r]], lv = labels[bv[r]];
        if (lu == r && lv != r) succ[r] = lv;
        else if (lv == r && lu != r) succ[r] = lu;
        else return -1;
    }
    int64_t *path = (int64_t *)malloc((size_t)(s > 0 ? s : 1) * sizeof(int64_t));
    for (int64_t i = 0; i < s; ++i) {
        int64_t r = reps[i];
        if (terminal[r] >= 0) continue;
        int64_t x = r, plen = 0, tval = -1, steps = 0;
        for (;;) {
            if (terminal[x] >= 0) { tval = terminal[x]; break; }
            int64_t y = succ[x];
            if (succ[y] == x) { tval = x < y ? x : y; terminal[x] = tval; terminal[y] = tval; break; }
            path[plen++] = x;
            x = y;
            if (++steps > s) { free(path); return -2; }
        }
        for (int64_t k = 0; k < plen; ++k) terminal[path[k]] = tval;
    }
    free(path);
    for (int64_t i = 0; i < s; ++i) {      /* ascending reps: first to reach a terminal is its minimum */
        int64_t tv = terminal[reps[i]];
        if (cluster_min[tv] < 0) cluster_min[tv] = reps[i];
    }
    for (int64_t i = 0; i < s; ++i) final_[reps[i]] = cluster_min[terminal[reps[i]]];
    int64_t ne = 0, nn = 0;
    for (int64_t i = 0; i < s; ++i) {
        int64_t r = reps[i], y = succ[r];
        if (!(succ[y] == r && y < r)) {    /* a mutual pair keeps its edge once */
            out_u[ne] = bu[r]; out_v[ne] = bv[r]; out_w[ne] = bw[r]; ++ne;
        }
        if (final_[r] == r) new_reps[nn++] = r;
    }
    *n_new = nn;
    return ne;
}

/* ---------------------------------------------------- per-phase exports */
/* Building blocks on reference-layout state, used to pin intermediate parity
 * (mst.py:436-547).  The tree is rebuilt from pts each call (cheap at test sizes). */

int oracle_reduce_labels(const float *pts, int64_t n, int d, const int64_t *labels, int64_t *il) {
    or_tree t;
    int rc = tree_build(&t, pts, n, d);
    if (rc) return rc;
    if (n > 1) reduce_labels(&t, labels, il);
    tree_free(&t);
    return OR_OK;
}

int oracle_upper_bounds(const float *pts, int64_t n, int d, const int64_t *perm, const int64_t *labels,
                        double *ub) {
    for (int64_t i = 0; i < n; ++i) ub[i] = INFINITY;   /* compute_upper_bounds resets all (mst.py:466) */
    upper_bounds(pts, d, perm, n, labels, NULL, ub);
    return OR_OK;
}

/* find_component_outgoing_edges (mst.py:472-514) with optional shard [q_begin, q_end)
 * of query slots (q_end <= 0 means all); best_* are n-sized, indexed by label. */
int oracle_find_edges(const float *pts, int64_t n, int d, const int64_t *labels, const int64_t *il,
                      const double *ub, int use_bounds, int skip, int64_t q_begin, int64_t q_end,
                      int64_t *best_u, int64_t *best_v, double *best_w, int64_t *evals) {
    or_tree t;
    int rc = tree_build(&t, pts, n, d);
    if (rc) return rc;
    int64_t *cu = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *cv = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    double *cw = (double *)malloc((size_t)n * sizeof(double));
    for (int64_t i = 0; i < n; ++i) { cu[i] = -1; cv[i] = -1; cw[i] = INFINITY;
                                      best_u[i] = -1; best_v[i] = -1; best_w[i] = INFINITY; }
    int ovf = 0;
    if (q_end <= 0) { q_begin = 0; q_end = n; }
    *evals = find_edges(&t, pts, labels, il, ub, NULL, use_bounds, skip, q_begin, q_end, cu, cv, cw, &ovf);
    reduce_candidates(labels, n, cu, cv, cw, best_u, best_v, best_w);
    free(cu); free(cv); free(cw);
    tree_free(&t);
    return ovf ? OR_ERR_STACK : OR_OK;
}

/* merge_components (mst.py:517-547); labels relabelled in place. */
int oracle_merge(int64_t n, const int64_t *reps, int64_t s, const int64_t *bu, const int64_t *bv,
                 const double *bw, int64_t *labels, int64_t *out_u, int64_t *out_v, double *out_w,
                 int64_t *n_edges, int64_t *new_reps, int64_t *n_new) {
    int64_t *succ = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *term = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *cmin = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *fin = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t ne = merge(reps, s, bu, bv, bw, labels, succ, term, cmin, fin, out_u, out_v, out_w, new_reps, n_new);
    int rc = OR_OK;
    if (ne == -1) rc = OR_ERR_NO_EDGE;
    else if (ne == -2) rc = OR_ERR_CHAIN;
    else if (*n_new >= s) rc = OR_ERR_NO_REDUCE;
    else for (int64_t i = 0; i < n; ++i) labels[i] = fin[labels[i]];
    *n_edges = ne;
    free(succ); free(term); free(cmin); free(fin);
    return rc;
}

/* ------------------------------------------------------------- the driver */

/* Final (w, u, v) order: equals np.lexsort((ev, eu, ew)) (mst.py:745-747).
 * LSD: v, then u, then the f64 bit pattern of w (w >= 0 so bits order like values). */
static int sort_edges(int64_t ne, const int64_t *eu, const int64_t *ev, const double *ew, int64_t *order) {
    uint64_t *key = (uint64_t *)malloc((size_t)(ne > 0 ? ne : 1) * sizeof(uint64_t));
    int64_t *tmp = (int64_t *)malloc((size_t)(ne > 0 ? ne : 1) * sizeof(int64_t));
    if (!key || !tmp) { free(key); free(tmp); return OR_ERR_ALLOC; }
    for (int64_t i = 0; i < ne; ++i) order[i] = i;
    int64_t *a = order, *b = tmp;
    for (int pass = 0; pass < 3; ++pass) {
        for (int64_t i = 0; i < ne; ++i) {
            if (pass == 0) key[i] = (uint64_t)ev[i];
            else if (pass == 1) key[i] = (uint64_t)eu[i];
            else { uint64_t bits; memcpy(&bits, &ew[i], 8); key[i] = bits; }
        }
        for (int shift = 0; shift < 64; shift += 16) {
            radix_pass(key, a, b, ne, shift);
            int64_t *t2 = a; a = b; b = t2;
        }
    }
    if (a != order) memcpy(order, a, (size_t)ne * sizeof(int64_t));
    free(key); free(tmp);
    return OR_OK;
}

typedef struct {
    int32_t iterations;
    int32_t num_counts;
    int64_t component_counts[64];
    int64_t leaf_distance_evals;
    double phase_seconds[8];   /* tree, core, reduce_labels, upper_bounds, find_edges, merge, mst, total */
} oracle_stats;

static double now_s(void) {
#ifdef _OPENMP
    return omp_get_wtime();
#else
    return 0.0;
#endif
}

/* (distance, index) order of the k-NN heap: 1 when entry 1 sorts after entry 2 (metric.py:87-91). */
static inline int heap_after(double d1, int64_t i1, double d2, int64_t i2) {
    return d1 > d2 || (d1 == d2 && i1 > i2);
}

/* Bounded max-heap push (metric.py:94-125); returns the new size. */
static int64_t heap_push(double *hd, int64_t *hi, int64_t size, int64_t k, double dd, int64_t p) {
    if (size < k) {
        int64_t i = size;
        hd[i] = dd; hi[i] = p;
        while (i > 0) {
            int64_t par = (i - 1) >> 1;
            if (heap_after(hd[i], hi[i], hd[par], hi[par])) {
                double td = hd[i]; hd[i] = hd[par]; hd[par] = td;
                int64_t ti = hi[i]; hi[i] = hi[par]; hi[par] = ti;
                i = par;
            } else break;
        }
        return size + 1;
    }
    if (heap_after(hd[0], hi[0], dd, p)) {
        hd[0] = dd; hi[0] = p;
        int64_t i = 0;
        for (;;) {
            int64_t l = 2 * i + 1, r = l + 1, big = i;
            if (l < size && heap_after(hd[l], hi[l], hd[big], hi[big])) big = l;
            if (r < size && heap_after(hd[r], hi[r], hd[big], hi[big])) big = r;
            if (big == i) break;
            double td = hd[i]; hd[i] = hd[big]; hd[big] = td;
            int64_t ti = hi[i]; hi[i] = hi[big]; hi[big] = ti;
            i = big;
        }
    }
    return size;
}

/* compute_core_distances (metric.py:128-234): per point the k-th nearest distance counting itself, one
 * bounded-radius traversal from the root with a (distance, index) max-heap of k entries; boxes at exactly
 * the radius are still visited.  out indexed by original point; k in [1, n]. */
static int core_distances(const or_tree *t, const float *pts, int64_t k, double *out) {
    const int64_t n = t->n, m = t->m;
    const int d = t->d;
    if (k == 1) { for (int64_t i = 0; i < n; ++i) out[i] = 0.0; return OR_OK; }
    int ovf = 0;
    #pragma omp parallel reduction(| : ovf)
    {
        double *hd = (double *)malloc((size_t)k * sizeof(double));
        int64_t *hi = (int64_t *)malloc((size_t)k * sizeof(int64_t));
        #pragma omp for schedule(dynamic, 1024)
        for (int64_t s = 0; s < n; ++s) {
            int64_t node_stack[OR_STACK];
            double dist_stack[OR_STACK];
            double q[3];
            int64_t qp = t->perm[s];
            for (int kk = 0; kk < d; ++kk) q[kk] = (double)pts[qp * d + kk];
            int64_t size = 0;
            double radius = INFINITY;
            node_stack[0] = 0;
            dist_stack[0] = m > 0 ? box_dist(t->box_lo, t->box_hi, d, 0, q) : 0.0;
            int top = m > 0 ? 1 : 0;
            if (m == 0) size = heap_push(hd, hi, size, k, 0.0, qp);
            while (top > 0) {
                --top;
                if (dist_stack[top] > radius) continue;
                int64_t ref = node_stack[top];
                int64_t child[2] = {t->left[ref], t->right[ref]};
                int64_t pa = -1, pb = -1;
                double pa_d = 0.0, pb_d = 0.0;
                for (int side = 0; side < 2; ++side) {
                    int64_t c = child[side];
                    if (c >= m) {
                        int64_t p = t->perm[c - m];
                        size = heap_push(hd, hi, size, k, point_dist(pts, d, p, q), p);
                        if (size == k) radius = hd[0];
                    } else {
                        double bd = box_dist(t->box_lo, t->box_hi, d, c, q);
                        if (bd <= radius) {
                            if (pa < 0) { pa = c; pa_d = bd; }
                            else { pb = c; pb_d = bd; }
                        }
                    }
                }
                if (pb >= 0) {
                    if (top + 2 > OR_STACK) { ovf = 1; top = 0; continue; }
                    if (pb_d < pa_d) {
                        int64_t tn = pa; pa = pb; pb = tn;
                        double td = pa_d; pa_d = pb_d; pb_d = td;
                    }
                    node_stack[top] = pb; dist_stack[top] = pb_d; ++top;
                    node_stack[top] = pa; dist_stack[top] = pa_d; ++top;
                } else if (pa >= 0) {
                    if (top + 1 > OR_STACK) { ovf = 1; top = 0; continue; }
                    node_stack[top] = pa; dist_stack[top] = pa_d; ++top;
                }
            }
            out[qp] = hd[0];
        }
        free(hd);
        free(hi);
    }
    return ovf ? OR_ERR_STACK : OR_OK;
}

int oracle_core_distances(const float *pts, int64_t n, int d, int64_t k, double *out) {
    or_tree t;
    int rc = tree_build(&t, pts, n, d);
    if (rc) return rc;
    rc = core_distances(&t, pts, k, out);
    tree_free(&t);
    return rc;
}

/* boruvka_emst / _run_boruvka, Euclidean metric (mst.py:578-769).
 * flags bit0 subtree_skip, bit1 upper_bound_seeding.  edges_out (n-1)x2 int64,
 * weights_out (n-1) float64, sorted by (w, u, v). */
static int boruvka(const float *pts, int64_t n, int d, int flags, int64_t k_pts, const double *given_cores,
                   int64_t *edges_out, double *weights_out, oracle_stats *st);

int oracle_boruvka(const float *pts, int64_t n, int d, int flags, int64_t *edges_out, double *weights_out,
                   oracle_stats *st) {
    return boruvka(pts, n, d, flags, 1, NULL, edges_out, weights_out, st);
}

/* boruvka_emst(points, "mrd", k_pts) / MutualReachability(core) (mst.py:638-644): given_cores (original
 * order) or NULL to compute them for k_pts (k_pts = 1 without a table is the Euclidean metric). */
int oracle_boruvka_mrd(const float *pts, int64_t n, int d, int flags, int64_t k_pts, const double *given_cores,
                       int64_t *edges_out, double *weights_out, oracle_stats *st) {
    return boruvka(pts, n, d, flags, k_pts, given_cores, edges_out, weights_out, st);
}

static int boruvka(const float *pts, int64_t n, int d, int flags, int64_t k_pts, const double *given_cores,
                   int64_t *edges_out, double *weights_out, oracle_stats *st) {
    const int skip = flags & 1, use_bounds = (flags >> 1) & 1;
    double t_start = now_s();
    memset(st, 0, sizeof(*st));
    or_tree t;
    int rc = tree_build(&t, pts, n, d);
    if (rc) return rc;
    double t_tree = now_s() - t_start;
    double tc = now_s();
    double *cores = NULL;
    if (given_cores || k_pts > 1) {
        cores = (double *)malloc((size_t)n * sizeof(double));
        if (!cores) { tree_free(&t); return OR_ERR_ALLOC; }
        if (given_cores) memcpy(cores, given_cores, (size_t)n * sizeof(double));
        else if ((rc = core_distances(&t, pts, k_pts, cores))) { free(cores); tree_free(&t); return rc; }
    }
    double t_core = now_s() - tc;
    double t0 = now_s();
    int64_t m = n - 1;
    int64_t *labels = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *il = (int64_t *)malloc((size_t)(m > 0 ? m : 1) * sizeof(int64_t));
    double *ub = (double *)malloc((size_t)n * sizeof(double));
    int64_t *reps = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *cu = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *cv = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    double *cw = (double *)malloc((size_t)n * sizeof(double));
    int64_t *bu = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *bv = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    double *bw = (double *)malloc((size_t)n * sizeof(double));
    int64_t *succ = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *term = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *cmin = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *fin = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *new_reps = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *eu = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *ev = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    double *ew = (double *)malloc((size_t)n * sizeof(double));
    int64_t *order = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    rc = OR_OK;
    if (!labels || !il || !ub || !reps || !cu || !cv || !cw || !bu || !bv || !bw || !succ || !term ||
        !cmin || !fin || !new_reps || !eu || !ev || !ew || !order) { rc = OR_ERR_ALLOC; goto done; }
    for (int64_t i = 0; i < n; ++i) { labels[i] = i; ub[i] = INFINITY; reps[i] = i; }
    for (int64_t i = 0; i < m; ++i) il[i] = OR_MIXED;
    int64_t nreps = n, ne_total = 0;
    int max_iters = 0;
    if (n > 1) { while (((int64_t)1 << max_iters) < n) ++max_iters; if (max_iters < 1) max_iters = 1; }
    st->component_counts[0] = n;
    st->num_counts = 1;
    double t_reduce = 0, t_bounds = 0, t_find = 0, t_merge = 0;
    while (nreps > 1) {
        st->iterations++;
        if (st->iterations > max_iters) { rc = OR_ERR_ITER; goto done; }
        double t1 = now_s();
        if (skip) reduce_labels(&t, labels, il);
        t_reduce += now_s() - t1;
        t1 = now_s();
        if (use_bounds) {
            for (int64_t i = 0; i < nreps; ++i) ub[reps[i]] = INFINITY;
            upper_bounds(pts, d, t.perm, n, labels, cores, ub);
        }
        t_bounds += now_s() - t1;
        t1 = now_s();
        int ovf = 0;
        st->leaf_distance_evals += find_edges(&t, pts, labels, il, ub, cores, use_bounds, skip, 0, n,
                                              cu, cv, cw, &ovf);
        if (ovf) { rc = OR_ERR_STACK; goto done; }
        for (int64_t i = 0; i < nreps; ++i) { bu[reps[i]] = -1; bv[reps[i]] = -1; bw[reps[i]] = INFINITY; }
        reduce_candidates(labels, n, cu, cv, cw, bu, bv, bw);
        t_find += now_s() - t1;
        t1 = now_s();
        int64_t nn = 0;
        int64_t ne = merge(reps, nreps, bu, bv, bw, labels, succ, term, cmin, fin,
                           eu + ne_total, ev + ne_total, ew + ne_total, new_reps, &nn);
        if (ne == -1) { rc = OR_ERR_NO_EDGE; goto done; }
        if (ne == -2) { rc = OR_ERR_CHAIN; goto done; }
        if (nn >= nreps) { rc = OR_ERR_NO_REDUCE; goto done; }
        #pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i) labels[i] = fin[labels[i]];
        ne_total += ne;
        memcpy(reps, new_reps, (size_t)nn * sizeof(int64_t));
        nreps = nn;
        if (st->num_counts < 64) st->component_counts[st->num_counts++] = nn;
        t_merge += now_s() - t1;
    }
    if (ne_total != n - 1) { rc = OR_ERR_COUNT; goto done; }
    rc = sort_edges(ne_total, eu, ev, ew, order);
    if (rc) goto done;
    for (int64_t i = 0; i < ne_total; ++i) {
        edges_out[2 * i] = eu[order[i]];
        edges_out[2 * i + 1] = ev[order[i]];
        weights_out[i] = ew[order[i]];
    }
    st->phase_seconds[0] = t_tree;
    st->phase_seconds[1] = t_core;
    st->phase_seconds[2] = t_reduce;
    st->phase_seconds[3] = t_bounds;
    st->phase_seconds[4] = t_find;
    st->phase_seconds[5] = t_merge;
    st->phase_seconds[6] = now_s() - t0;
    st->phase_seconds[7] = now_s() - t_start;
done:
    free(labels); free(il); free(ub); free(reps); free(cu); free(cv); free(cw); free(bu); free(bv); free(bw);
    free(succ); free(term); free(cmin); free(fin); free(new_reps); free(eu); free(ev); free(ew); free(order);
    free(cores);
    tree_free(&t);
    return rc;
}
