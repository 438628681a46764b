"""ctypes front-end of the CPU oracle (``oracle/emst_oracle.c``).

TEST INFRASTRUCTURE ONLY -- the parity checker and the reported CPU baseline.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its cpu_baseline
and ``--impl reference`` legs) may import this module.  The product package
``paper_2207_00514_b200`` never imports it and has no CPU fallback.

The C restatement follows the reference package function by function
(/root/reference/pkg/src/emst/{geometry,bvh,mst}.py; citations in the C file) and
is pinned against golden vectors recorded from the reference itself
(tests/golden/make_goldens.py, tests/test_oracle_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle_emst.so")

_ERRORS = {
    1: "TraversalStackOverflowError",
    2: "InternalInvariantViolation: a component found no valid outgoing edge",
    3: "InternalInvariantViolation: component chain did not terminate in a pair",
    4: "InternalInvariantViolation: merge did not reduce the component count",
    5: "InternalInvariantViolation: iteration bound exceeded",
    6: "InternalInvariantViolation: edge count mismatch",
    7: "allocation failure",
    8: "InternalInvariantViolation: hierarchy topology",
}

_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")


class _Stats(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int32),
        ("num_counts", ctypes.c_int32),
        ("component_counts", ctypes.c_int64 * 64),
        ("leaf_distance_evals", ctypes.c_int64),
        ("phase_seconds", ctypes.c_double * 8),
    ]


_lib = None


def build() -> str:
    """Compile the oracle with its Makefile (gcc + OpenMP)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        i64, i32 = ctypes.c_int64, ctypes.c_int
        L.oracle_morton_codes.argtypes = [_f32p, i64, i32, _u64p]
        L.oracle_morton_codes.restype = None
        L.oracle_sort_by_morton.argtypes = [_f32p, i64, i32, _i64p]
        L.oracle_sort_by_morton.restype = None
        L.oracle_build.argtypes = [_f32p, i64, i32, _i64p, _i64p, _i64p, _i64p, _i64p, _f32p, _f32p]
        L.oracle_reduce_labels.argtypes = [_f32p, i64, i32, _i64p, _i64p]
        L.oracle_upper_bounds.argtypes = [_f32p, i64, i32, _i64p, _i64p, _f64p]
        L.oracle_find_edges.argtypes = [_f32p, i64, i32, _i64p, _i64p, _f64p, i32, i32, i64, i64,
                                        _i64p, _i64p, _f64p, ctypes.POINTER(ctypes.c_int64)]
        L.oracle_merge.argtypes = [i64, _i64p, i64, _i64p, _i64p, _f64p, _i64p, _i64p, _i64p, _f64p,
                                   ctypes.POINTER(ctypes.c_int64), _i64p, ctypes.POINTER(ctypes.c_int64)]
        L.oracle_boruvka.argtypes = [_f32p, i64, i32, i32, _i64p, _f64p, ctypes.POINTER(_Stats)]
        L.oracle_boruvka_mrd.argtypes = [_f32p, i64, i32, i32, i64, ctypes.c_void_p, _i64p, _f64p,
                                         ctypes.POINTER(_Stats)]
        L.oracle_core_distances.argtypes = [_f32p, i64, i32, i64, _f64p]
        L.oracle_num_threads.restype = ctypes.c_int
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def _pts(points) -> np.ndarray:
    return np.ascontiguousarray(points, dtype=np.float32)


def _check(rc: int):
    if rc:
        raise RuntimeError(f"oracle error {rc}: {_ERRORS.get(rc, 'unknown')}")


def num_threads() -> int:
    return lib().oracle_num_threads()


def set_threads(t: int) -> None:
    lib().oracle_set_threads(int(t))


def morton_codes(points) -> np.ndarray:
    p = _pts(points)
    out = np.empty(p.shape[0], np.uint64)
    lib().oracle_morton_codes(p, p.shape[0], p.shape[1], out)
    return out


def sort_by_morton(points) -> np.ndarray:
    p = _pts(points)
    out = np.empty(p.shape[0], np.int64)
    lib().oracle_sort_by_morton(p, p.shape[0], p.shape[1], out)
    return out


@dataclass
class OracleTree:
    perm: np.ndarray
    left: np.ndarray
    right: np.ndarray
    parent: np.ndarray
    leaf_parent: np.ndarray
    box_lo: np.ndarray
    box_hi: np.ndarray


def build_tree(points) -> OracleTree:
    p = _pts(points)
    n, d = p.shape
    m = max(n - 1, 0)
    t = OracleTree(np.empty(n, np.int64), np.empty(m, np.int64), np.empty(m, np.int64),
                   np.empty(m, np.int64), np.empty(n, np.int64), np.empty((m, d), np.float32),
                   np.empty((m, d), np.float32))
    # ndpointer rejects zero-size (m == 0) arrays only if None; give 1-element buffers then
    bufs = [a if a.size else np.empty(1, a.dtype) for a in
            (t.left, t.right, t.parent, t.box_lo, t.box_hi)]
    _check(lib().oracle_build(p, n, d, t.perm, bufs[0], bufs[1], bufs[2], t.leaf_parent,
                              bufs[3].reshape(-1), bufs[4].reshape(-1)))
    return t


def reduce_labels(points, labels) -> np.ndarray:
    p = _pts(points)
    n = p.shape[0]
    il = np.full(max(n - 1, 1), -1, np.int64)
    _check(lib().oracle_reduce_labels(p, n, p.shape[1], np.ascontiguousarray(labels, np.int64), il))
    return il[: max(n - 1, 0)]


def upper_bounds(points, perm, labels) -> np.ndarray:
    p = _pts(points)
    ub = np.empty(p.shape[0], np.float64)
    _check(lib().oracle_upper_bounds(p, p.shape[0], p.shape[1], np.ascontiguousarray(perm, np.int64),
                                     np.ascontiguousarray(labels, np.int64), ub))
    return ub


def find_edges(points, labels, internal_labels, ub, *, use_bounds=True, skip=True, q_begin=0, q_end=0):
    """Per-component best (u, v, w) arrays indexed by label, plus leaf evals."""
    p = _pts(points)
    n = p.shape[0]
    bu = np.empty(n, np.int64)
    bv = np.empty(n, np.int64)
    bw = np.empty(n, np.float64)
    ev = ctypes.c_int64(0)
    il = np.ascontiguousarray(internal_labels, np.int64)
    if il.size == 0:
        il = np.full(1, -1, np.int64)
    _check(lib().oracle_find_edges(p, n, p.shape[1], np.ascontiguousarray(labels, np.int64), il,
                                   np.ascontiguousarray(ub, np.float64), int(use_bounds), int(skip),
                                   int(q_begin), int(q_end), bu, bv, bw, ctypes.byref(ev)))
    return bu, bv, bw, ev.value


def merge(labels, reps, bu, bv, bw):
    """Returns (labels_out, edge_u, edge_v, edge_w, new_reps)."""
    lab = np.array(labels, dtype=np.int64, copy=True)
    reps = np.ascontiguousarray(reps, np.int64)
    s = reps.shape[0]
    ou = np.empty(max(s, 1), np.int64)
    ov = np.empty(max(s, 1), np.int64)
    ow = np.empty(max(s, 1), np.float64)
    nr = np.empty(max(s, 1), np.int64)
    ne = ctypes.c_int64(0)
    nn = ctypes.c_int64(0)
    _check(lib().oracle_merge(lab.shape[0], reps, s, np.ascontiguousarray(bu, np.int64),
                              np.ascontiguousarray(bv, np.int64), np.ascontiguousarray(bw, np.float64),
                              lab, ou, ov, ow, ctypes.byref(ne), nr, ctypes.byref(nn)))
    return lab, ou[: ne.value], ov[: ne.value], ow[: ne.value], nr[: nn.value]


@dataclass
class OracleResult:
    edges: np.ndarray
    weights: np.ndarray
    total_weight: float
    iterations: int
    component_counts: list = field(default_factory=list)
    leaf_distance_evals: int = 0
    phase_timings: dict = field(default_factory=dict)


PHASES = ("tree", "core", "reduce_labels", "upper_bounds", "find_edges", "merge", "mst", "total")


def core_distances(points, k_pts: int) -> np.ndarray:
    """compute_core_distances (metric.py:128-234): k_pts-th nearest distance counting self, by point."""
    p = _pts(points)
    n, d = p.shape
    out = np.empty(n, np.float64)
    _check(lib().oracle_core_distances(p, n, d, int(k_pts), out))
    return out


def boruvka_emst(points, *, subtree_skip=True, upper_bound_seeding=True, k_pts: int = 1,
                 cores=None) -> OracleResult:
    """The reference's boruvka_emst (mst.py:578-769): Euclidean, or mutual reachability when k_pts > 1
    (cores computed as compute_core_distances) or a core table is given (MutualReachability)."""
    p = _pts(points)
    n, d = p.shape
    edges = np.empty((max(n - 1, 1), 2), np.int64)
    weights = np.empty(max(n - 1, 1), np.float64)
    st = _Stats()
    flags = (1 if subtree_skip else 0) | (2 if upper_bound_seeding else 0)
    if cores is None and k_pts == 1:
        _check(lib().oracle_boruvka(p, n, d, flags, edges.reshape(-1), weights, ctypes.byref(st)))
    else:
        c = None if cores is None else np.ascontiguousarray(cores, np.float64)
        _check(lib().oracle_boruvka_mrd(p, n, d, flags, int(k_pts), None if c is None else c.ctypes.data,
                                        edges.reshape(-1), weights, ctypes.byref(st)))
    edges = edges[: n - 1]
    weights = weights[: n - 1]
    return OracleResult(
        edges=edges, weights=weights, total_weight=float(np.sum(weights)),
        iterations=int(st.iterations),
        component_counts=[int(st.component_counts[i]) for i in range(st.num_counts)],
        leaf_distance_evals=int(st.leaf_distance_evals),
        phase_timings={k: float(st.phase_seconds[i]) for i, k in enumerate(PHASES)},
    )
