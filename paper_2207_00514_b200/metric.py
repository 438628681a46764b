"""Edge-weight metrics: Euclidean and mutual reachability (reference pkg/src/emst/metric.py).

Mutual reachability weights a pair by max(core(u), core(v), d(u, v)), where
core(p) is the distance from p to its k_pts-th nearest neighbour counting p
itself (metric.py:1-8).  The GPU path computes core distances with the same
climb traversal as the edge search (csrc/core.cuh) and threads them through
the bound seeding and the traversal; k_pts = 1 is plain Euclidean bit for bit.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import DimensionMismatchError, InvalidIndexError, InvalidParameterError
from .geometry import as_point_array, distance


@dataclass(frozen=True)
class Euclidean:
    """Plain Euclidean distance (metric.py:30-32)."""


@dataclass(frozen=True)
class CoreDistances:
    """Distance from each point to its k_pts-th nearest neighbour, self included (metric.py:35-45).

    values[i] is indexed by original point index; k_pts = 1 gives all zeros.
    """

    k_pts: int
    values: np.ndarray


@dataclass(frozen=True)
class MutualReachability:
    """max(core(u), core(v), Euclidean(u, v)) for a fixed core table (metric.py:48-52)."""

    core: CoreDistances


def core_array(metric, n: int) -> np.ndarray:
    """Per-point core distances for a metric: zeros for Euclidean (metric.py:58-70)."""
    if isinstance(metric, Euclidean):
        return np.zeros(n, dtype=np.float64)
    if isinstance(metric, MutualReachability):
        values = np.ascontiguousarray(metric.core.values, dtype=np.float64)
        if values.shape != (n,):
            raise DimensionMismatchError(f"core table has {values.shape[0]} entries for {n} points")
        return values
    raise InvalidParameterError(f"unknown metric {metric!r}")


def edge_weight(metric, u: int, v: int, points) -> float:
    """Weight of the edge (u, v) under a metric (metric.py:73-84)."""
    pts = as_point_array(points)
    n = pts.shape[0]
    for idx in (u, v):
        if not 0 <= idx < n:
            raise InvalidIndexError(f"point index {idx} out of range for {n} points")
    base = distance(pts[u], pts[v])
    if isinstance(metric, Euclidean):
        return base
    cores = core_array(metric, n)
    return max(base, float(cores[u]), float(cores[v]))


def compute_core_distances(bvh, points, k_pts: int) -> CoreDistances:
    """k_pts-th nearest-neighbour distance of every point, self included (metric.py:209-234), on the GPU.

    Exact f64 distances in the reference's arithmetic; the value is the k-th
    smallest of the distances to all points (p itself at 0, duplicates at 0).
    """
    pts = as_point_array(points)
    n = pts.shape[0]
    if pts.shape[0] != bvh.num_points or pts.shape[1] != bvh.dim:
        raise DimensionMismatchError("points array does not match the hierarchy")
    if not isinstance(k_pts, (int, np.integer)) or isinstance(k_pts, bool):
        raise InvalidParameterError(f"k_pts must be an integer, got {k_pts!r}")
    k = int(k_pts)
    if k < 1 or k > n:
        raise InvalidParameterError(f"k_pts must be in [1, {n}], got {k}")
    if k == 1:
        return CoreDistances(1, np.zeros(n, dtype=np.float64))
    out = np.empty(n, dtype=np.float64)
    ctx = _lib.default_context()
    e = _lib.err_buf()
    with ctx.lock:
        rc = _lib.load().emst_core_distances(ctx.handle, pts.ctypes.data, n, pts.shape[1], 0, k,
                                             out.ctypes.data, e, len(e))
    _lib.raise_for(rc, e)
    return CoreDistances(k, out)


def core_pointer(metric, n: int):
    """(keep-alive array, ctypes pointer) of a metric's core table for the C ABI; (None, None) for Euclidean."""
    if metric is None or isinstance(metric, Euclidean):
        return None, None
    values = core_array(metric, n)
    return values, values.ctypes.data
