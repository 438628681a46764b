"""LBVH over Morton-sorted points, built on the GPU (drop-in for pkg/src/emst/bvh.py).

``build`` runs the sm_100a pipeline (scene bounds, Morton codes, onesweep radix
sort, Karras topology, atomic-arrival refit) and returns the tree in the
reference's array layout (bvh.py:39-75): same node numbering, same leaf order,
same boxes -- tests/test_gpu_parity.py compares them array for array.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import (
    DimensionMismatchError,
    InvalidCoordinateError,
    InvalidIndexError,
    InvalidParameterError,
    TraversalStackOverflowError,
    UnsupportedDimensionError,
)
from .geometry import Aabb, as_point_array, check_shape

STACK_CAPACITY = 64   # bvh.py:36


@dataclass
class Bvh:
    """Flat arrays of one hierarchy (bvh.py:39-109).

    leaf_perm[s] is the original index of Z-order slot s; left/right hold packed
    child refs (< n - 1 internal, >= n - 1 leaf slot + n - 1); the root is node 0.
    """

    num_points: int
    dim: int
    leaf_perm: np.ndarray
    left: np.ndarray
    right: np.ndarray
    parent: np.ndarray
    leaf_parent: np.ndarray
    box_lo: np.ndarray
    box_hi: np.ndarray
    # bottom-up level schedule (bvh.py:60-63): nodes sweep_order[sweep_starts[k]:sweep_starts[k + 1]]
    # have height k + 1
    sweep_order: np.ndarray | None = None
    sweep_starts: np.ndarray | None = None
    # the points the GPU built this tree from (the building blocks rebuild from them)
    points: np.ndarray | None = field(default=None, repr=False, compare=False)
    # the native context that still holds this tree on the device, and the token naming it there:
    # the building blocks reuse it instead of rebuilding while the token is current
    tree_context: object = field(default=None, repr=False, compare=False)
    tree_token: int = field(default=0, repr=False, compare=False)

    @property
    def num_internal(self) -> int:
        return self.num_points - 1

    @property
    def num_nodes(self) -> int:
        return 2 * self.num_points - 1

    @property
    def root(self) -> int:
        return 0

    def is_leaf_ref(self, ref: int) -> bool:
        return ref >= self.num_internal

    def leaf_slot(self, ref: int) -> int:
        if not self.is_leaf_ref(ref):
            raise InvalidIndexError(f"ref {ref} is an internal node")
        return ref - self.num_internal

    def leaf_ref(self, slot: int) -> int:
        if not 0 <= slot < self.num_points:
            raise InvalidIndexError(f"leaf slot {slot} out of range")
        return self.num_internal + slot

    def node_box(self, internal_index: int) -> Aabb:
        if not 0 <= internal_index < self.num_internal:
            raise InvalidIndexError(f"internal node {internal_index} out of range")
        return Aabb(self.box_lo[internal_index].astype(np.float64), self.box_hi[internal_index].astype(np.float64))


def _device_points(points):
    """(pointer, n, d, flags, keepalive) for numpy input or a CUDA float32 tensor."""
    try:
        import torch
        if isinstance(points, torch.Tensor) and points.is_cuda:
            if points.dtype != torch.float32:
                points = points.float()
            points = points.contiguous()
            n, d = check_shape(points)
            return points.data_ptr(), n, d, _lib.POINTS_ON_DEVICE, points
    except ImportError:
        pass
    arr = np.asarray(points)
    if arr.dtype == np.float32 and arr.ndim == 2 and arr.flags.c_contiguous:
        # already in the device layout: the finiteness check (and the reference's
        # "point {row} has a non-finite coordinate" error) runs on the GPU in k_scene
        n, d = check_shape(arr)
        return arr.ctypes.data, n, d, 0, arr
    pts = as_point_array(arr)
    n, d = pts.shape
    return pts.ctypes.data, n, d, 0, pts


def _is_cuda_tensor(x) -> bool:
    try:
        import torch
    except ImportError:
        return False
    return isinstance(x, torch.Tensor) and x.is_cuda


def context_for(keep, context=None) -> _lib.Context:
    """The native context a call runs on, ordered after the stream that produced `keep`.

    A CUDA tensor goes to a context on its own device (the default one for that
    device unless `context` is given, which must then be on the same device), and
    the context's stream first waits for torch's current stream there: the
    tensor (or the float32 / contiguous copy _device_points made of it) may
    still be in flight.  Host input uses the current device's default context.
    """
    if _is_cuda_tensor(keep):
        ctx = context if context is not None else _lib.default_context(keep.device.index)
        ctx.after_torch(keep)
        return ctx
    return context if context is not None else _lib.default_context()


def _bounds_arrays(bounds: Aabb | None, d: int):
    """(keep-alive, lo pointer, hi pointer) of an Aabb for the C ABI; NULLs for the tight scene box."""
    if bounds is None:
        return None, None, None
    if not isinstance(bounds, Aabb):
        raise InvalidParameterError(f"bounds must be an Aabb, got {type(bounds).__name__}")
    if bounds.dim != d:
        raise DimensionMismatchError("bounds dimension differs from point dimension")
    lo = np.ascontiguousarray(bounds.lo, np.float64)
    hi = np.ascontiguousarray(bounds.hi, np.float64)
    return (lo, hi), lo.ctypes.data, hi.ctypes.data


def morton_codes(points, bounds: Aabb | None = None) -> np.ndarray:
    """Morton codes quantised against `bounds` (the tight scene box by default), on the GPU
    (geometry.py:209-227): 63 bits in 3D, 62 in 2D; points outside `bounds` are clamped into it."""
    p, n, d, flags, keep = _device_points(points)
    bkeep, blo, bhi = _bounds_arrays(bounds, d)
    out = np.empty(n, np.uint64)
    ctx = context_for(keep)
    e = _lib.err_buf()
    with ctx.lock:
        rc = _lib.load().emst_morton_codes(ctx.handle, p, n, d, flags, blo, bhi, out.ctypes.data, e, len(e))
    _lib.raise_for(rc, e)
    return out


def morton_encode(point, bounds: Aabb) -> int:
    """Morton code of one point within `bounds`, clamped into it (geometry.py:230-244)."""
    p = np.asarray(point, dtype=np.float64)
    if p.ndim != 1:
        raise UnsupportedDimensionError("morton_encode takes a single point")
    if p.shape[0] != bounds.dim:
        raise DimensionMismatchError("point dimension differs from bounds dimension")
    if not np.isfinite(p).all():
        raise InvalidCoordinateError("point has a non-finite coordinate")
    return int(morton_codes(p.astype(np.float32)[None, :], bounds)[0])


def sort_by_morton(points, bounds: Aabb | None = None) -> np.ndarray:
    """Permutation ordering the points by (Morton code, original index) (geometry.py:247-254): the
    solve's stable onesweep radix sort on the GPU."""
    p, n, d, flags, keep = _device_points(points)
    bkeep, blo, bhi = _bounds_arrays(bounds, d)
    out = np.empty(n, np.int64)
    ctx = context_for(keep)
    e = _lib.err_buf()
    with ctx.lock:
        rc = _lib.load().emst_sort_by_morton(ctx.handle, p, n, d, flags, blo, bhi, out.ctypes.data, e, len(e))
    _lib.raise_for(rc, e)
    return out


def build(points) -> Bvh:
    """Build the hierarchy on the GPU and return it in the reference layout (bvh.py:305-340)."""
    p, n, d, flags, keep = _device_points(points)
    m = n - 1
    perm = np.empty(n, np.int64)
    left = np.empty(max(m, 1), np.int64)
    right = np.empty(max(m, 1), np.int64)
    parent = np.empty(max(m, 1), np.int64)
    leaf_parent = np.empty(n, np.int64)
    box_lo = np.empty((max(m, 1), d), np.float32)
    box_hi = np.empty((max(m, 1), d), np.float32)
    order = np.empty(max(m, 1), np.int64)
    starts = np.empty(n, np.int64)
    n_starts = ctypes.c_int64(0)
    ctx = context_for(keep)
    e = _lib.err_buf()
    with ctx.lock:
        rc = _lib.load().emst_build(ctx.handle, p, n, d, flags, perm.ctypes.data, left.ctypes.data, right.ctypes.data,
                                    parent.ctypes.data, leaf_parent.ctypes.data, box_lo.ctypes.data,
                                    box_hi.ctypes.data, order.ctypes.data, starts.ctypes.data,
                                    ctypes.byref(n_starts), e, len(e))
    _lib.raise_for(rc, e)
    host = keep if isinstance(keep, np.ndarray) else keep.detach().cpu().numpy()
    token = ctx.tree_token()
    ctx.tree_points = (token, points, host)   # (compute_upper_bounds names points, not a Bvh)
    return Bvh(n, d, perm, left[:m], right[:m], parent[:m], leaf_parent, box_lo[:m], box_hi[:m], order[:m],
               starts[:n_starts.value].copy(), host, ctx, token)


def _ref_bound(bvh: Bvh, coords: np.ndarray, q: np.ndarray, ref: int) -> float:
    """f64 distance from q to a leaf point (ref >= n - 1) or to an internal node's box, axes summed in
    order without fused operations (bvh.py:267-290)."""
    m = bvh.num_internal
    acc = 0.0
    if ref >= m:
        p = coords[int(bvh.leaf_perm[ref - m])]
        for k in range(bvh.dim):
            g = float(q[k]) - float(p[k])
            acc += g * g
    else:
        lo, hi = bvh.box_lo[ref], bvh.box_hi[ref]
        for k in range(bvh.dim):
            x = float(q[k])
            g = float(lo[k]) - x if x < float(lo[k]) else (x - float(hi[k]) if x > float(hi[k]) else 0.0)
            acc += g * g
    return math.sqrt(acc)


def traverse_nearest(bvh: Bvh, points, query, *, on_leaf, prune=None, radius: float = math.inf) -> float:
    """Constrained nearest-neighbour walk from the root with caller callbacks (bvh.py:343-418).

    Host-side: the callbacks are arbitrary Python, so this walk runs on the CPU over the
    GPU-built arrays (the solve's own traversal never comes here).  Same contract as the
    reference: depth first, nearer child first (the left one on a tie), ``on_leaf(point, dist)``
    may return a smaller radius, ``prune(ref, lower_bound, radius)`` may veto an entry (default:
    drop it when lower_bound > radius), at most STACK_CAPACITY entries stacked.
    """
    coords = as_point_array(points)
    if coords.shape != (bvh.num_points, bvh.dim):
        raise DimensionMismatchError("points array does not match the hierarchy")
    q = np.asarray(query, dtype=np.float64)
    if q.shape != (bvh.dim,):
        raise DimensionMismatchError("query dimension differs from hierarchy dimension")
    m = bvh.num_internal
    start = 0 if m > 0 else m   # one point: the root is the leaf itself
    pending = [(start, _ref_bound(bvh, coords, q, start))]
    while pending:
        ref, lb = pending.pop()
        veto = prune(ref, lb, radius) if prune is not None else lb > radius
        if veto:
            continue
        if ref >= m:
            got = on_leaf(int(bvh.leaf_perm[ref - m]), lb)
            if got is not None:
                radius = float(got)
            continue
        kids = [(int(bvh.left[ref]), 0), (int(bvh.right[ref]), 1)]
        bounds = [(_ref_bound(bvh, coords, q, c), side, c) for c, side in kids]
        bounds.sort()   # nearer first; equal bounds keep the left child nearer
        if len(pending) + 2 > STACK_CAPACITY:
            raise TraversalStackOverflowError(f"traversal exceeded {STACK_CAPACITY} stacked nodes")
        for b, _, c in reversed(bounds):   # the nearer one ends on top
            pending.append((c, b))
    return radius


def for_each_leaf_to_root(bvh: Bvh, visit) -> None:
    """Bottom-up rendezvous over the internal nodes (bvh.py:421-440): every leaf climbs; the first
    arrival at a node stops, the second calls ``visit(node)`` (so a node is visited once, after both
    subtrees) and climbs on unless ``visit`` returned False.  Host-side, for caller callbacks; the
    GPU's refit and height kernels run the same protocol with atomics."""
    seen = np.zeros(bvh.num_internal, dtype=bool)
    for slot in range(bvh.num_points):
        node = int(bvh.leaf_parent[slot])
        while node >= 0:
            if not seen[node]:
                seen[node] = True
                break
            if visit(node) is False:
                break
            node = int(bvh.parent[node])
