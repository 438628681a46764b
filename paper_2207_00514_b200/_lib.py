"""ctypes binding of the native library ``libemst_b200.so`` (C ABI: include/emst_b200.h).

There is no CPU fallback: if the library is missing, fails to load, or no CUDA
device is present, every compute call raises :class:`~.errors.DeviceError`.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

from .errors import (
    DeviceError,
    EmptyDatasetError,
    InternalInvariantViolation,
    InvalidCoordinateError,
    InvalidParameterError,
    NoOutgoingEdgeError,
    NothingToFindError,
    TraversalStackOverflowError,
    UnsupportedDimensionError,
)

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EMST_LIB_PATH") or os.path.join(PKG_DIR, "libemst_b200.so")
CSRC = os.path.join(PKG_DIR, "csrc")

SUBTREE_SKIP = 1
UPPER_BOUNDS = 2
POINTS_ON_DEVICE = 4
OUTPUT_ON_DEVICE = 8

PHASES = ("tree", "core", "reduce_labels", "upper_bounds", "find_edges", "merge", "mst", "total")

# emst_status -> exception class (include/emst_b200.h)
_STATUS = {
    1: EmptyDatasetError,
    2: UnsupportedDimensionError,
    3: InvalidCoordinateError,
    4: TraversalStackOverflowError,
    5: InternalInvariantViolation,
    6: InternalInvariantViolation,
    7: InternalInvariantViolation,
    8: InternalInvariantViolation,
    9: InternalInvariantViolation,
    10: DeviceError,
    11: DeviceError,
    12: InvalidParameterError,
    13: InvalidParameterError,
    14: NothingToFindError,
    15: NoOutgoingEdgeError,
}


class Stats(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int32),
        ("num_counts", ctypes.c_int32),
        ("component_counts", ctypes.c_int64 * 64),
        ("leaf_distance_evals", ctypes.c_int64),
        ("phase_ms", ctypes.c_double * 8),
        ("bad_row", ctypes.c_int64),
        ("kernel_launches", ctypes.c_int64),
        ("h2d_bytes", ctypes.c_int64),
        ("d2h_bytes", ctypes.c_int64),
        ("world", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("traverse_ms", ctypes.c_double),
        ("traverse_launches", ctypes.c_int64),
        ("traverse_queries", ctypes.c_int64),
        ("round_traverse_ms", ctypes.c_double * 64),
        ("round_node_visits", ctypes.c_int64 * 64),
        ("round_found", ctypes.c_int64 * 64),
        ("round_skipped", ctypes.c_int64 * 64),
        ("total_weight", ctypes.c_double),
        ("host_in_ms", ctypes.c_double),
        ("host_out_ms", ctypes.c_double),
    ]


EXPORTS = (
    "emst_nccl_unique_id",
    "emst_context_create",
    "emst_context_destroy",
    "emst_context_set_stream",
    "emst_context_set_virtual_shards",
    "emst_context_set_exchange",
    "emst_context_wait_stream",
    "emst_tree_token",
    "emst_context_reuse_tree",
    "emst_context_set_state_on_device",
    "emst_boruvka",
    "emst_boruvka_mrd",
    "emst_core_distances",
    "emst_morton_codes",
    "emst_sort_by_morton",
    "emst_build",
    "emst_reduce_labels",
    "emst_compute_upper_bounds",
    "emst_find_component_outgoing_edges",
    "emst_merge_components",
    "emst_format_edges",
    "emst_format_points",
    "emst_text_free",
    "emst_count_rows",
    "emst_parse_rows",
    "emst_build_info",
)

# int (*)(uint64_t* buf, int64_t count, int32_t op, void* user): in-place all-reduce over the ranks
EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p)
EXCHANGE_MIN, EXCHANGE_SUM = 0, 1

_lib = None
_lock = threading.Lock()


def build(verbose: bool = False) -> str:
    """Compile the CUDA library in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
    cmd = ["make", "-C", CSRC]
    if not verbose:
        cmd.insert(1, "-s")
    subprocess.run(cmd, check=True)
    return LIB_PATH


def load():
    """Load and type the native library (raises DeviceError if it is absent)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise DeviceError(f"native library {LIB_PATH} is missing; run __graft_entry__.build() "
                              "(make -C paper_2207_00514_b200/csrc)")
        try:
            L = ctypes.CDLL(LIB_PATH)
        except OSError as exc:
            raise DeviceError(f"cannot load {LIB_PATH}: {exc}") from exc
        vp, i64, i32, cp, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_char_p, ctypes.c_size_t
        L.emst_nccl_unique_id.argtypes = [vp, cp, sz]
        L.emst_context_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, ctypes.POINTER(vp), cp, sz]
        L.emst_context_destroy.argtypes = [vp]
        L.emst_context_set_virtual_shards.argtypes = [vp, ctypes.c_int]
        L.emst_context_set_stream.argtypes = [vp, vp]
        L.emst_context_set_exchange.argtypes = [vp, EXCHANGE_FN, vp]
        L.emst_context_wait_stream.argtypes = [vp, vp]
        L.emst_tree_token.argtypes = [vp, ctypes.POINTER(i64)]
        L.emst_context_reuse_tree.argtypes = [vp, i64]
        L.emst_context_set_state_on_device.argtypes = [vp, ctypes.c_int]
        L.emst_boruvka.argtypes = [vp, vp, i64, i32, i32, vp, vp, ctypes.POINTER(Stats), cp, sz]
        L.emst_boruvka_mrd.argtypes = [vp, vp, i64, i32, i32, i64, vp, vp, vp, ctypes.POINTER(Stats), cp, sz]
        L.emst_core_distances.argtypes = [vp, vp, i64, i32, i32, i64, vp, cp, sz]
        L.emst_morton_codes.argtypes = [vp, vp, i64, i32, i32, vp, vp, vp, cp, sz]
        L.emst_sort_by_morton.argtypes = [vp, vp, i64, i32, i32, vp, vp, vp, cp, sz]
        L.emst_build.argtypes = [vp, vp, i64, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, cp, sz]
        L.emst_reduce_labels.argtypes = [vp, vp, i64, i32, vp, vp, cp, sz]
        L.emst_compute_upper_bounds.argtypes = [vp, vp, i64, i32, vp, vp, vp, cp, sz]
        L.emst_find_component_outgoing_edges.argtypes = [vp, vp, i64, i32, vp, vp, vp, i32, vp, vp, vp, vp, cp, sz]
        L.emst_merge_components.argtypes = [vp, i64, vp, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, cp, sz]
        L.emst_format_edges.argtypes = [vp, vp, i64, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(i64)]
        L.emst_format_points.argtypes = [vp, i64, i32, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(i64)]
        L.emst_text_free.argtypes = []
        L.emst_count_rows.argtypes = [vp, i64, ctypes.POINTER(i64)]
        L.emst_parse_rows.argtypes = [vp, i64, i64, i64, i64, i32, i32, vp, vp, i64, vp]
        for name in EXPORTS:
            getattr(L, name).restype = ctypes.c_int
        L.emst_build_info.restype = ctypes.c_char_p
        L.emst_text_free.restype = None
        _lib = L
        return L


def raise_for(code: int, err: ctypes.Array, stats: Stats | None = None):
    if code == 0:
        return
    msg = err.value.decode(errors="replace") if err is not None else f"status {code}"
    exc = _STATUS.get(code, DeviceError)
    raise exc(msg)


def err_buf():
    return ctypes.create_string_buffer(512)


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data


class Context:
    """One native context: a CUDA device, its stream and workspace, optionally an NCCL rank."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: bytes | None = None):
        L = load()
        h = ctypes.c_void_p()
        e = err_buf()
        idbuf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        rc = L.emst_context_create(int(device), int(rank), int(world), idbuf, ctypes.byref(h), e, len(e))
        raise_for(rc, e)
        self.handle = h
        self.device, self.rank, self.world = int(device), int(rank), int(world)
        self.lock = threading.Lock()

    def set_virtual_shards(self, shards: int) -> None:
        rc = load().emst_context_set_virtual_shards(self.handle, int(shards))
        if rc == 11:
            raise DeviceError("cannot create the 1-rank NCCL communicator for virtual shards")
        if rc:
            raise InvalidParameterError(f"virtual shard count {shards} out of range [1, 64]")

    def set_exchange(self, allreduce) -> None:
        """Host exchange for a world > 1 context made without an NCCL id.

        ``allreduce(buf, op)`` gets a numpy uint64 view of page-locked host
        memory and must all-reduce it in place over every rank: unsigned min
        for ``op == EXCHANGE_MIN``, sum for ``EXCHANGE_SUM``.
        """
        def _cb(buf, count, op, user):
            try:
                arr = np.ctypeslib.as_array((ctypes.c_uint64 * int(count)).from_address(buf)) if count else \
                    np.empty(0, np.uint64)
                allreduce(arr, int(op))
                return 0
            except Exception as exc:   # (an exception cannot cross the C frame)
                self.exchange_error = exc
                return 1
        self._exchange_cb = EXCHANGE_FN(_cb)   # keep the thunk alive with the context
        self.exchange_error = None
        raise_for(load().emst_context_set_exchange(self.handle, self._exchange_cb, None), None)

    def wait_stream(self, stream) -> None:
        """Order this context's stream after the work queued on ``stream`` (torch.cuda.Stream or raw handle)."""
        handle = getattr(stream, "cuda_stream", stream)
        rc = load().emst_context_wait_stream(self.handle, ctypes.c_void_p(handle) if handle else None)
        if rc:
            raise DeviceError(f"cudaStreamWaitEvent failed (status {rc})")

    def after_torch(self, tensor) -> None:
        """Before handing the library a CUDA tensor: wait for torch's current stream on its device, which
        may still be producing it (the context runs on its own non-blocking stream)."""
        import torch
        if tensor.device.index != self.device:
            raise InvalidParameterError(f"tensor on cuda:{tensor.device.index} given to a cuda:{self.device} context")
        self.wait_stream(torch.cuda.current_stream(tensor.device))

    def tree_token(self) -> int:
        """Names the tree this context holds now (0: none); every build changes it."""
        t = ctypes.c_int64(0)
        raise_for(load().emst_tree_token(self.handle, ctypes.byref(t)), None)
        return int(t.value)

    def reuse_tree(self, token: int) -> None:
        """The next building-block call skips its build if `token` still names this context's tree."""
        raise_for(load().emst_context_reuse_tree(self.handle, int(token)), None)

    def state_on_device(self, on: bool) -> None:
        """While on, the building blocks take and return device pointers for the round state."""
        raise_for(load().emst_context_set_state_on_device(self.handle, 1 if on else 0), None)

    def set_stream(self, stream) -> None:
        """Run on an external CUDA stream (a torch.cuda.Stream or a raw cudaStream_t int; None = own)."""
        handle = getattr(stream, "cuda_stream", stream)
        load().emst_context_set_stream(self.handle, ctypes.c_void_p(handle) if handle else None)

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            load().emst_context_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    L = load()
    buf = ctypes.create_string_buffer(128)
    e = err_buf()
    raise_for(L.emst_nccl_unique_id(buf, e, len(e)), e)
    return buf.raw


_default: dict[int, Context] = {}


def default_context(device: int | None = None) -> Context:
    """Process-wide single-GPU context for `device` (current CUDA device by default)."""
    if device is None:
        device = _current_device()
    with _lock:
        ctx = _default.get(device)
    if ctx is None:
        ctx = Context(device)
        with _lock:
            _default.setdefault(device, ctx)
            ctx = _default[device]
    return ctx


def set_default_context(ctx: Context) -> None:
    with _lock:
        _default[ctx.device] = ctx


def _current_device() -> int:
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:
        pass
    return 0
