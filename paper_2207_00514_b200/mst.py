"""The drop-in entry point: ``boruvka_emst`` on a B200 (pkg/src/emst/mst.py:578-769).

Same signature, validation order, exceptions and ``MstResult`` as the
reference.  The work happens in ``libemst_b200.so``: every phase of the
single-tree Boruvka loop is a hand-written sm_100a kernel;
this module only validates arguments, hands the points over (host numpy array
or a CUDA float32 tensor, zero-copy) and wraps the outputs.

The per-round building blocks (``reduce_labels``, ``compute_upper_bounds``,
``find_component_outgoing_edges``, ``merge_components``; mst.py:436-547) are
exported too, each backed by the same GPU kernels the loop uses.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .bvh import Bvh, _device_points, context_for
from .errors import (
    DimensionMismatchError,
    InternalInvariantViolation,
    InvalidParameterError,
    NoOutgoingEdgeError,
    NothingToFindError,
)
from .geometry import as_point_array
from .metric import CoreDistances, Euclidean, MutualReachability, core_array, core_pointer

MIXED = -1   # mst.py:57


@dataclass(frozen=True)
class WeightedEdge:
    """Undirected edge with canonical u < v, ordered by (weight, u, v) (mst.py:62-89)."""

    u: int
    v: int
    weight: float

    def __post_init__(self):
        if self.u == self.v:
            raise InvalidParameterError(f"self edge at {self.u}")
        if self.u < 0 or self.v < 0:
            raise InvalidParameterError("edge endpoints must be non-negative")
        if self.u > self.v:
            lo, hi = self.v, self.u
            object.__setattr__(self, "u", lo)
            object.__setattr__(self, "v", hi)

    @property
    def key(self) -> tuple[float, int, int]:
        return (self.weight, self.u, self.v)

    def __lt__(self, other: "WeightedEdge") -> bool:
        return self.key < other.key


@dataclass
class ComponentState:
    """Per-point representative labels, internal-node labels and radii (mst.py:92-117)."""

    labels: np.ndarray
    internal_labels: np.ndarray
    upper_bounds: np.ndarray

    @classmethod
    def initial(cls, bvh: Bvh, device=None) -> "ComponentState":
        """Every point its own component.  ``device`` (e.g. "cuda") keeps the state in HBM as torch
        tensors: the building blocks then run round after round without host copies."""
        n = bvh.num_points
        if device is not None:
            import torch
            dev = torch.device(device)
            return cls(torch.arange(n, dtype=torch.int64, device=dev),
                       torch.full((max(n - 1, 0),), MIXED, dtype=torch.int64, device=dev),
                       torch.full((n,), math.inf, dtype=torch.float64, device=dev))
        return cls(np.arange(n, dtype=np.int64), np.full(max(n - 1, 0), MIXED, dtype=np.int64),
                   np.full(n, np.inf, dtype=np.float64))

    @property
    def num_components(self) -> int:
        if _on_device(self.labels):
            return int(_device_reps(self.labels).numel())
        return int(np.unique(self.labels).shape[0])


@dataclass
class OutgoingEdges:
    """Cheapest outgoing edge per live component; u, v, w indexed by representative (mst.py:120-137)."""

    reps: np.ndarray
    u: np.ndarray
    v: np.ndarray
    w: np.ndarray
    leaf_distance_evals: int

    def edge(self, rep: int) -> WeightedEdge:
        if self.v[rep] < 0:
            raise NoOutgoingEdgeError(f"component {rep} has no recorded edge")
        return WeightedEdge(int(self.u[rep]), int(self.v[rep]), float(self.w[rep]))


@dataclass
class MergeOutcome:
    """One iteration's collapse of the component graph (mst.py:140-155)."""

    num_components: int
    edge_u: np.ndarray
    edge_v: np.ndarray
    edge_w: np.ndarray
    new_reps: np.ndarray

    @property
    def edges(self) -> list[WeightedEdge]:
        return [WeightedEdge(int(u), int(v), float(w)) for u, v, w in zip(self.edge_u, self.edge_v, self.edge_w)]


@dataclass
class MstResult:
    """A spanning tree plus run instrumentation (mst.py:158-182).

    edges (n-1, 2) int64 with u < v, rows sorted by (weight, u, v); weights
    aligned float64; phase_timings in seconds (device-timed phases, host-timed
    total); component_counts from n down to 1.
    """

    edges: np.ndarray
    weights: np.ndarray
    total_weight: float
    iterations: int
    phase_timings: dict = field(default_factory=dict)
    component_counts: list = field(default_factory=list)
    leaf_distance_evals: int = 0
    threads: int = 1
    kernel_launches: int = 0
    gpus: int = 1

    def edge_list(self) -> list[WeightedEdge]:
        return [WeightedEdge(int(u), int(v), float(w)) for (u, v), w in zip(self.edges, self.weights)]


def _resolve_threads(threads) -> int:
    """Validated like mst.py:550-559; the GPU build reports one host thread."""
    if not isinstance(threads, (int, np.integer)):
        raise InvalidParameterError(f"threads must be an integer, got {threads!r}")
    if int(threads) < 0:
        raise InvalidParameterError(f"threads must be >= 0, got {int(threads)}")
    return 1


def _resolve_metric(metric) -> tuple[str, CoreDistances | None]:
    """(kind, given core table) as mst.py:562-575."""
    if isinstance(metric, str):
        name = metric.strip().lower().replace("_", "-")
        if name == "euclidean":
            return "euclidean", None
        if name in ("mrd", "mutual-reachability"):
            return "mrd", None
        raise InvalidParameterError(f"metric must be 'euclidean' or 'mrd', got {metric!r}")
    if isinstance(metric, Euclidean):
        return "euclidean", None
    if isinstance(metric, MutualReachability):
        return "mrd", metric.core
    raise InvalidParameterError(f"unknown metric {metric!r}")


def _raise_call(rc: int, e, ctx: _lib.Context) -> None:
    """raise_for, re-raising a host-exchange callback's own exception first."""
    err = getattr(ctx, "exchange_error", None)
    if rc and err is not None:
        ctx.exchange_error = None
        raise err
    _lib.raise_for(rc, e)


def _host_outputs(m: int):
    """(m, 2) int64 and (m,) float64 host arrays for the results.

    Page-locked when torch is present (its caching host allocator recycles the
    pages across calls, and the device->host copy runs at full PCIe/C2C rate
    instead of faulting in fresh pageable memory); plain numpy otherwise.
    """
    try:
        import torch
        if torch.cuda.is_available():
            e = torch.empty((m, 2), dtype=torch.int64, pin_memory=True).numpy()
            w = torch.empty((m,), dtype=torch.float64, pin_memory=True).numpy()
            return e, w
    except Exception:
        pass
    return np.empty((m, 2), np.int64), np.empty(m, np.float64)


def boruvka_emst(points, metric="euclidean", k_pts: int = 1, *, threads: int = 0, subtree_skip: bool = True,
                 upper_bound_seeding: bool = True, context: _lib.Context | None = None) -> MstResult:
    """Euclidean minimum spanning tree of (n, d) points, d in {2, 3}, on the GPU.

    Drop-in for the reference's ``boruvka_emst`` (mst.py:578-624): identical
    edges and weights (bit for bit, including ties), iterations and
    component_counts.  ``points`` may be array-like (copied host -> device) or a
    CUDA float32 tensor (used in place).  ``context`` selects a device / NCCL
    rank set up by :mod:`.distributed`; by default the current device's.
    """
    t_start = time.perf_counter()
    if not isinstance(k_pts, (int, np.integer)) or isinstance(k_pts, bool):
        raise InvalidParameterError(f"k_pts must be an integer, got {k_pts!r}")
    k_pts = int(k_pts)
    if k_pts < 1:
        raise InvalidParameterError(f"k_pts must be >= 1, got {k_pts}")
    kind, given_core = _resolve_metric(metric)
    if kind == "euclidean" and k_pts != 1:
        raise InvalidParameterError("k_pts applies to the mrd metric only")
    nthreads = _resolve_threads(threads)

    p, n, d, flags, keep = _device_points(points)
    core_keep, core_ptr = None, None
    if kind == "mrd":
        # mst.py:638-644: a given table (shape-checked by core_array), else k_pts in [1, n]
        if given_core is not None:
            core_keep = core_array(MutualReachability(given_core), n)
            core_ptr = core_keep.ctypes.data
        elif k_pts > n:
            raise InvalidParameterError(f"k_pts must be in [1, {n}], got {k_pts}")
    flags |= (_lib.SUBTREE_SKIP if subtree_skip else 0) | (_lib.UPPER_BOUNDS if upper_bound_seeding else 0)
    ne = n - 1
    edges, weights = _host_outputs(max(ne, 1))
    st = _lib.Stats()
    ctx = context_for(keep, context)
    e = _lib.err_buf()
    with ctx.lock:
        if kind == "mrd":
            rc = _lib.load().emst_boruvka_mrd(ctx.handle, p, n, d, flags, k_pts, core_ptr, edges.ctypes.data,
                                              weights.ctypes.data, ctypes.byref(st), e, len(e))
        else:
            rc = _lib.load().emst_boruvka(ctx.handle, p, n, d, flags, edges.ctypes.data, weights.ctypes.data,
                                          ctypes.byref(st), e, len(e))
    ctx.last_stats = st
    _raise_call(rc, e, ctx)
    edges = edges[:ne]
    weights = weights[:ne]
    total = time.perf_counter() - t_start
    timings = {k: st.phase_ms[i] / 1e3 for i, k in enumerate(_lib.PHASES)}
    timings["total"] = max(total, timings["tree"] + timings["core"] + timings["mst"])
    return MstResult(
        edges=edges,
        weights=weights,
        # float(np.sum(weights)) (mst.py:749), summed on the device in numpy's pairwise order
        total_weight=float(st.total_weight) if ne > 0 else 0.0,
        iterations=int(st.iterations),
        phase_timings=timings,
        component_counts=[int(st.component_counts[i]) for i in range(st.num_counts)],
        leaf_distance_evals=int(st.leaf_distance_evals),
        threads=nthreads,
        kernel_launches=int(st.kernel_launches),
        gpus=int(st.world),
    )


# ----------------------------------------------------- per-round building blocks
# Each call runs on the native context that holds the Bvh's tree when there is
# one (no rebuild while its token is current), and on device-resident state when
# the state's arrays are CUDA tensors (ComponentState.initial(bvh, device="cuda")):
# then nothing crosses PCIe but a few counters.

def _on_device(x) -> bool:
    try:
        import torch
    except ImportError:
        return False
    return isinstance(x, torch.Tensor) and x.is_cuda


def _device_reps(labels):
    """np.unique of device labels (values in [0, n)) without a sort.  The reference's labels name a
    member of their component that labels itself (its smallest index), so the representatives are
    the fixed points i == labels[i] -- checked by one gather (labels[labels] == labels); anything
    else goes through torch.unique."""
    import torch
    n = labels.shape[0]
    if n == 0:
        return labels.new_empty(0)
    lo, hi = torch.aminmax(labels)
    if int(lo) < 0 or int(hi) >= n:
        raise InvalidParameterError(f"labels must lie in [0, {n})")
    if bool(torch.equal(labels[labels], labels)):
        return torch.nonzero(labels == torch.arange(n, device=labels.device)).view(-1)
    return torch.unique(labels)


def _dev_array(x, dtype_name: str, n: int, what: str):
    """A contiguous CUDA tensor of `dtype_name` and length n (the device-state contract)."""
    import torch
    dt = getattr(torch, dtype_name)
    if not _on_device(x) or x.dtype != dt or x.dim() != 1 or x.shape[0] != n:
        raise DimensionMismatchError(f"{what} must be a CUDA {dtype_name} vector of length {n}")
    return x if x.is_contiguous() else x.contiguous()


class _Call:
    """Context, tree reuse and state location for one building-block call."""

    def __init__(self, bvh: Bvh | None, points, state):
        self.device_state = _on_device(state.labels)
        if self.device_state:
            dev = state.labels.device.index
            ctx = bvh.tree_context if bvh is not None and getattr(bvh.tree_context, "device", None) == dev else None
            self.ctx = ctx if ctx is not None else _lib.default_context(dev)
            self.ctx.after_torch(state.labels)
        else:
            ctx = bvh.tree_context if bvh is not None else None
            self.ctx = ctx if ctx is not None else _lib.default_context()
        # (token, points given to build(), the float32 array the tree was built from), set by build()
        held = getattr(self.ctx, "tree_points", None)
        self.token = 0
        if bvh is not None and bvh.tree_context is self.ctx:
            if points is None or points is bvh.points or (held is not None and held[0] == bvh.tree_token
                                                          and held[1] is points):
                self.token = bvh.tree_token
        elif bvh is None and points is not None and held is not None and (held[1] is points or held[2] is points):
            self.token = held[0]

    def points(self, points):
        """(keep-alive, pointer, n, d) of the points the call hands over.  With the tree reused they were
        validated when it was built and are not read again: only their shape is checked."""
        if self.token:
            shape = tuple(points.shape) if hasattr(points, "shape") else np.asarray(points).shape
            if len(shape) != 2:
                raise DimensionMismatchError("points must be a 2-D array")
            return None, None, int(shape[0]), int(shape[1])
        pts = as_point_array(points)
        return pts, pts.ctypes.data, pts.shape[0], pts.shape[1]

    def __enter__(self):
        self.ctx.lock.acquire()
        if self.token:
            self.ctx.reuse_tree(self.token)
        self.ctx.state_on_device(self.device_state)
        return self

    def __exit__(self, *exc):
        self.ctx.state_on_device(False)
        self.ctx.reuse_tree(0)
        self.ctx.lock.release()


def reduce_labels(bvh: Bvh, state: ComponentState):
    """Internal-node labels, MIXED where children disagree (mst.py:436-448).

    The GPU derives node labels from slot-range boundary counts over the tree it
    built for ``bvh`` (reused while it is the context's current tree, else rebuilt
    from ``bvh.points``).
    """
    if state.labels.shape[0] != bvh.num_points:
        raise DimensionMismatchError("state does not match the hierarchy")
    if bvh.points is None:
        raise InvalidParameterError("reduce_labels needs a Bvh produced by build() (it carries its points)")
    n = bvh.num_points
    if n > 1:
        call = _Call(bvh, None, state)
        pts, pp, n, d = call.points(bvh.points)
        e = _lib.err_buf()
        if call.device_state:
            lab = _dev_array(state.labels, "int64", n, "labels")
            out = _dev_array(state.internal_labels, "int64", n - 1, "internal_labels")
            lp, op = lab.data_ptr(), out.data_ptr()
        else:
            lab = np.ascontiguousarray(state.labels, np.int64)
            out = np.empty(n - 1, np.int64)
            lp, op = lab.ctypes.data, out.ctypes.data
        with call:
            rc = _lib.load().emst_reduce_labels(call.ctx.handle, pp, n, d, lp, op, e, len(e))
        _lib.raise_for(rc, e)
        if out is not state.internal_labels:
            state.internal_labels[:] = out
    return state.internal_labels


def compute_upper_bounds(state: ComponentState, z_order, points, metric=None):
    """Seed radii from Z-adjacent cross-component pairs (mst.py:451-469)."""
    call = _Call(None, points, state)
    pts, pp, n, d = call.points(points)
    if state.labels.shape[0] != n or len(z_order) != n:
        raise DimensionMismatchError("state, order, and points disagree on size")
    core_keep, core_ptr = core_pointer(metric, n)
    e = _lib.err_buf()
    if call.device_state:
        lab = _dev_array(state.labels, "int64", n, "labels")
        ub = _dev_array(state.upper_bounds, "float64", n, "upper_bounds")
        lp, up = lab.data_ptr(), ub.data_ptr()
    else:
        lab = np.ascontiguousarray(state.labels, np.int64)
        ub = np.empty(n, np.float64)
        lp, up = lab.ctypes.data, ub.ctypes.data
    with call:
        rc = _lib.load().emst_compute_upper_bounds(call.ctx.handle, pp, n, d, lp, core_ptr, up, e, len(e))
    _lib.raise_for(rc, e)
    if ub is not state.upper_bounds:
        state.upper_bounds[:] = ub
    return state.upper_bounds


def find_component_outgoing_edges(bvh: Bvh, points, state: ComponentState, metric=None, *,
                                  subtree_skip: bool = True, use_upper_bounds: bool = True) -> OutgoingEdges:
    """Cheapest edge leaving every live component (mst.py:472-514)."""
    call = _Call(bvh, points, state)
    pts, pp, n, d = call.points(points)
    if state.labels.shape[0] != n or d != bvh.dim or bvh.num_points != n:
        raise DimensionMismatchError("state does not match the hierarchy")
    flags = (_lib.SUBTREE_SKIP if subtree_skip else 0) | (_lib.UPPER_BOUNDS if use_upper_bounds else 0)
    core_keep, core_ptr = core_pointer(metric, n)
    evals = ctypes.c_int64(0)
    e = _lib.err_buf()
    if call.device_state:
        import torch
        lab = _dev_array(state.labels, "int64", n, "labels")
        ub = _dev_array(state.upper_bounds, "float64", n, "upper_bounds")
        reps = _device_reps(lab)
        if reps.numel() < 2:
            raise NothingToFindError("a single component has no outgoing edges")
        bu = torch.empty(n, dtype=torch.int64, device=lab.device)
        bv = torch.empty_like(bu)
        bw = torch.empty(n, dtype=torch.float64, device=lab.device)
        ptrs = (lab.data_ptr(), ub.data_ptr(), bu.data_ptr(), bv.data_ptr(), bw.data_ptr())
    else:
        reps = np.unique(state.labels).astype(np.int64)
        if reps.shape[0] < 2:
            raise NothingToFindError("a single component has no outgoing edges")
        lab = np.ascontiguousarray(state.labels, np.int64)
        ub = np.ascontiguousarray(state.upper_bounds, np.float64)
        bu = np.empty(n, np.int64)
        bv = np.empty(n, np.int64)
        bw = np.empty(n, np.float64)
        ptrs = (lab.ctypes.data, ub.ctypes.data, bu.ctypes.data, bv.ctypes.data, bw.ctypes.data)
    with call:
        rc = _lib.load().emst_find_component_outgoing_edges(
            call.ctx.handle, pp, n, d, ptrs[0], ptrs[1], core_ptr, flags,
            ptrs[2], ptrs[3], ptrs[4], ctypes.byref(evals), e, len(e))
    _lib.raise_for(rc, e)
    missing = reps[bv[reps] < 0]
    if missing.shape[0] > 0:
        raise NoOutgoingEdgeError(f"component {int(missing[0])} found no outgoing edge")
    return OutgoingEdges(reps, bu, bv, bw, int(evals.value))


def merge_components(state: ComponentState, outgoing: OutgoingEdges) -> MergeOutcome:
    """Collapse the chosen-edge graph; relabel in place (mst.py:517-547)."""
    n = state.labels.shape[0]
    call = _Call(None, None, state)
    ne = ctypes.c_int64(0)
    nn = ctypes.c_int64(0)
    e = _lib.err_buf()
    if call.device_state:
        import torch
        s = int(outgoing.reps.shape[0])
        reps = _dev_array(outgoing.reps, "int64", s, "reps")
        lab = _dev_array(state.labels, "int64", n, "labels")
        bu = _dev_array(outgoing.u, "int64", n, "u")
        bv = _dev_array(outgoing.v, "int64", n, "v")
        bw = _dev_array(outgoing.w, "float64", n, "w")
        dev = lab.device
        ou = torch.empty(max(s, 1), dtype=torch.int64, device=dev)
        ov = torch.empty_like(ou)
        ow = torch.empty(max(s, 1), dtype=torch.float64, device=dev)
        nr = torch.empty_like(ou)
        ptrs = [t.data_ptr() for t in (reps, bu, bv, bw, lab, ou, ov, ow, nr)]
    else:
        reps = np.ascontiguousarray(outgoing.reps, np.int64)
        s = reps.shape[0]
        lab = np.ascontiguousarray(state.labels, np.int64).copy()
        ou = np.empty(max(s, 1), np.int64)
        ov = np.empty(max(s, 1), np.int64)
        ow = np.empty(max(s, 1), np.float64)
        nr = np.empty(max(s, 1), np.int64)
        bu = np.ascontiguousarray(outgoing.u, np.int64)
        bv = np.ascontiguousarray(outgoing.v, np.int64)
        bw = np.ascontiguousarray(outgoing.w, np.float64)
        ptrs = [a.ctypes.data for a in (reps, bu, bv, bw, lab, ou, ov, ow, nr)]
    with call:
        rc = _lib.load().emst_merge_components(call.ctx.handle, n, ptrs[0], s, ptrs[1], ptrs[2], ptrs[3], ptrs[4],
                                               ptrs[5], ptrs[6], ptrs[7], ctypes.byref(ne), ptrs[8],
                                               ctypes.byref(nn), e, len(e))
    if rc == 5:
        raise InternalInvariantViolation("a component's chosen edge is inconsistent")
    _lib.raise_for(rc, e)
    if lab is not state.labels:
        state.labels[:] = lab
    k, m = ne.value, nn.value
    return MergeOutcome(int(m), ou[:k].clone() if call.device_state else ou[:k].copy(),
                        ov[:k].clone() if call.device_state else ov[:k].copy(),
                        ow[:k].clone() if call.device_state else ow[:k].copy(),
                        nr[:m].clone() if call.device_state else nr[:m].copy())


def iteration_bound(n: int) -> int:
    """ceil(log2 n) Boruvka rounds at most (mst.py:671)."""
    return max(1, math.ceil(math.log2(n))) if n > 1 else 0


def boruvka_emst_device(points, edges_out, weights_out, *, subtree_skip: bool = True,
                        upper_bound_seeding: bool = True, context: _lib.Context | None = None) -> _lib.Stats:
    """Device-resident variant: CUDA float32 points in, results written into CUDA tensors.

    ``edges_out`` is an (n-1, 2) int64 CUDA tensor and ``weights_out`` an (n-1,)
    float64 CUDA tensor; nothing crosses PCIe but the per-round control words.
    Returns the raw run statistics.  Used by bench.py for the HBM-resident number.
    """
    import torch

    if not (isinstance(points, torch.Tensor) and points.is_cuda and points.dtype == torch.float32):
        raise InvalidParameterError("points must be a CUDA float32 tensor")
    pts = points.contiguous()
    if pts.ndim != 2:
        raise DimensionMismatchError(f"points must be (n, d), got shape {tuple(pts.shape)}")
    n, d = int(pts.shape[0]), int(pts.shape[1])
    for name, t, dtype, shape in (("edges_out", edges_out, torch.int64, (max(n - 1, 0), 2)),
                                  ("weights_out", weights_out, torch.float64, (max(n - 1, 0),))):
        if not isinstance(t, torch.Tensor) or t.dtype != dtype or not t.is_cuda:
            raise InvalidParameterError(f"{name} must be a CUDA {dtype} tensor")
        if t.device != pts.device:
            raise InvalidParameterError(f"{name} is on {t.device}, the points on {pts.device}")
        if tuple(t.shape) != shape:
            raise DimensionMismatchError(f"{name} must have shape {shape}, got {tuple(t.shape)}")
        if not t.is_contiguous():
            raise InvalidParameterError(f"{name} must be contiguous")
    flags = _lib.POINTS_ON_DEVICE | _lib.OUTPUT_ON_DEVICE
    flags |= (_lib.SUBTREE_SKIP if subtree_skip else 0) | (_lib.UPPER_BOUNDS if upper_bound_seeding else 0)
    st = _lib.Stats()
    ctx = context_for(pts, context)
    # the outputs may have been allocated (or still be read) on torch's stream: covered by the same wait
    e = _lib.err_buf()
    with ctx.lock:
        rc = _lib.load().emst_boruvka(ctx.handle, pts.data_ptr(), n, d, flags, edges_out.data_ptr(),
                                      weights_out.data_ptr(), ctypes.byref(st), e, len(e))
    _raise_call(rc, e, ctx)
    return st
