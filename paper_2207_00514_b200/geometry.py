"""Input validation, boxes and distances (host side of pkg/src/emst/geometry.py).

Only validation and the scalar helpers live here; Morton codes and the Z-order
sort run on the GPU (csrc/build.cu) and are exposed through :mod:`.bvh`.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import (
    DimensionMismatchError,
    EmptyDatasetError,
    InvalidCoordinateError,
    UnsupportedDimensionError,
)

MORTON_BITS_2D = 31   # geometry.py:28
MORTON_BITS_3D = 21   # geometry.py:29


def check_shape(arr) -> tuple[int, int]:
    """ndim / n / d checks of as_point_array, in the reference's order (geometry.py:58-67)."""
    if arr.ndim != 2:
        raise UnsupportedDimensionError(f"expected a 2-dimensional (n, d) array, got ndim={arr.ndim}")
    n, d = arr.shape
    if n == 0:
        raise EmptyDatasetError("point set is empty")
    if d not in (2, 3):
        raise UnsupportedDimensionError(f"points must have 2 or 3 coordinates, got {d}")
    return int(n), int(d)


def nonfinite_error(row: int) -> InvalidCoordinateError:
    return InvalidCoordinateError(f"point {row} has a non-finite coordinate")


def as_point_array(points) -> np.ndarray:
    """Validate and normalise to a C-contiguous (n, d) float32 array (geometry.py:36-71)."""
    arr = np.asarray(points)
    check_shape(arr)
    finite = np.isfinite(arr)
    if not finite.all():
        raise nonfinite_error(int(np.flatnonzero(~finite.all(axis=1))[0]))
    return np.ascontiguousarray(arr, dtype=np.float32)


@dataclass(frozen=True)
class Aabb:
    """Axis-aligned box with inclusive float64 corners (geometry.py:74-99)."""

    lo: np.ndarray
    hi: np.ndarray

    def __post_init__(self):
        lo = np.asarray(self.lo, dtype=np.float64)
        hi = np.asarray(self.hi, dtype=np.float64)
        if lo.shape != hi.shape or lo.ndim != 1:
            raise DimensionMismatchError("box corners must be 1-d arrays of equal length")
        if np.any(lo > hi):
            raise InvalidCoordinateError("box has lo > hi on some axis")
        object.__setattr__(self, "lo", lo)
        object.__setattr__(self, "hi", hi)

    @property
    def dim(self) -> int:
        return self.lo.shape[0]

    def contains(self, point) -> bool:
        p = np.asarray(point, dtype=np.float64)
        if p.shape != self.lo.shape:
            raise DimensionMismatchError("point dimension differs from box dimension")
        return bool(np.all(p >= self.lo) and np.all(p <= self.hi))


def scene_bounds(points) -> Aabb:
    """Tight inclusive box of a non-empty point set (geometry.py:102-105)."""
    pts = as_point_array(points)
    return Aabb(pts.min(axis=0).astype(np.float64), pts.max(axis=0).astype(np.float64))


def distance(u, v) -> float:
    """Euclidean distance in float64, axes summed in order (geometry.py:108-124)."""
    a = np.asarray(u, dtype=np.float64)
    b = np.asarray(v, dtype=np.float64)
    if a.shape != b.shape or a.ndim != 1:
        raise DimensionMismatchError(
            f"distance needs two points of equal dimension, got {a.shape} and {b.shape}")
    acc = 0.0
    for k in range(a.shape[0]):
        diff = float(a[k]) - float(b[k])
        acc += diff * diff
    return math.sqrt(acc)


def distance_point_box(point, box: Aabb) -> float:
    """Distance from a point to a box, 0 inside (geometry.py:127-140)."""
    p = np.asarray(point, dtype=np.float64)
    if p.shape != box.lo.shape:
        raise DimensionMismatchError("point dimension differs from box dimension")
    acc = 0.0
    for k in range(p.shape[0]):
        x, lo, hi = float(p[k]), float(box.lo[k]), float(box.hi[k])
        gap = lo - x if x < lo else (x - hi if x > hi else 0.0)
        acc += gap * gap
    return math.sqrt(acc)
