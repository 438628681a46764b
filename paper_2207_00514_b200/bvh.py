"""LBVH over Morton-sorted points, built on the GPU (drop-in for pkg/src/emst/bvh.py).

``build`` runs the sm_100a pipeline (scene bounds, Morton codes, onesweep radix
sort, Karras topology, atomic-arrival refit) and returns the tree in the
reference's array layout (bvh.py:39-75): same node numbering, same leaf order,
same boxes -- tests/test_gpu_parity.py compares them array for array.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import InvalidIndexError
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
    # the points the GPU built this tree from (the building blocks rebuild from them)
    points: np.ndarray | None = field(default=None, repr=False, compare=False)

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


def morton_codes(points) -> np.ndarray:
    """Morton codes with the tight scene bounds, computed on the GPU (geometry.py:209-227)."""
    p, n, d, flags, keep = _device_points(points)
    out = np.empty(n, np.uint64)
    ctx = context_for(keep)
    e = _lib.err_buf()
    with ctx.lock:
        rc = _lib.load().emst_morton_codes(ctx.handle, p, n, d, flags, out.ctypes.data, e, len(e))
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
    ctx = context_for(keep)
    e = _lib.err_buf()
    with ctx.lock:
        rc = _lib.load().emst_build(ctx.handle, p, n, d, flags, perm.ctypes.data, left.ctypes.data, right.ctypes.data,
                                    parent.ctypes.data, leaf_parent.ctypes.data, box_lo.ctypes.data,
                                    box_hi.ctypes.data, e, len(e))
    _lib.raise_for(rc, e)
    host = keep if isinstance(keep, np.ndarray) else keep.detach().cpu().numpy()
    return Bvh(n, d, perm, left[:m], right[:m], parent[:m], leaf_parent, box_lo[:m], box_hi[:m], host)


def sort_by_morton(points) -> np.ndarray:
    """Z-order permutation with index tie-break (geometry.py:247-254), from the GPU sort."""
    return build(points).leaf_perm
