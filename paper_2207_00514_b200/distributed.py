"""Multi-GPU plumbing: one process per GPU, torch.distributed for the rendezvous.

The tree is replicated (every rank builds the same one from the same points,
deterministically), each Boruvka round's traversal is split by Morton slot
range -- the reference's ``prange`` over query blocks (mst.py:236) cut into
``world`` contiguous pieces -- and the per-component minima meet in a
two-phase min all-reduce issued by the native library:

  phase A  all-reduce-min of the f64 weight bit patterns, one u64 per component;
  phase B  all-reduce-min of (u << 32 | v) over the ranks whose local weight
           equals the global one (all-ones elsewhere).

u64 min on the bit pattern of a non-negative double is the numeric min, and
phase B then picks the smallest (u, v) among the minimum-weight candidates, so
the pair of u64 reductions is exactly the reference's 128-bit (w, u, v) order
(mst.py:62-89) -- a single u64 all-reduce of a truncated key would not be.

Two transports carry the all-reduce, both behind the same device kernels
(k_split_keys / k_mask_uv / k_join_keys in csrc/boruvka.cuh):

  * ``"nccl"``: the library's own NCCL communicator (ncclAllReduce on its
    stream, over NVLink/NVSwitch); torch.distributed only carries the 128-byte
    unique id from rank 0 to the others.
  * ``"host"``: a callback into torch.distributed.all_reduce on page-locked
    host copies -- any backend (gloo), any device placement, including several
    ranks sharing one GPU (which NCCL refuses).  The multi-rank parity tests
    use it to run the real N-rank path on a single-GPU machine.
"""

from __future__ import annotations

import os

import numpy as np

from . import _lib

_SIGN = np.uint64(1 << 63)


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Morton slot range [begin, end) of `rank`'s queries (same formula as the C++ side)."""
    return rank * n // world, (rank + 1) * n // world


def broadcast_nccl_id(group=None) -> bytes:
    """Create the NCCL unique id on rank 0 and hand it to every rank of `group`."""
    import torch.distributed as dist

    obj = [_lib.nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return obj[0]


def host_allreduce(group=None):
    """The host exchange: ``f(buf, op)`` all-reduces a numpy uint64 array in place over `group`.

    torch has no unsigned 64-bit reduction, so min runs on int64 after flipping
    the sign bit (x ^ 2^63 maps unsigned order onto signed order, the all-ones
    "no edge" key included); sum runs on the int64 view (wrap-around is the
    same bits).
    """
    import torch
    import torch.distributed as dist

    def allreduce(buf: np.ndarray, op: int) -> None:
        if op == _lib.EXCHANGE_MIN:
            t = torch.from_numpy((buf ^ _SIGN).view(np.int64))
            dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
            buf[:] = t.numpy().view(np.uint64) ^ _SIGN
        elif op == _lib.EXCHANGE_SUM:
            t = torch.from_numpy(buf.view(np.int64).copy())
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
            buf[:] = t.numpy().view(np.uint64)
        else:
            raise ValueError(f"unknown exchange op {op}")

    return allreduce


def init_context(group=None, device: int | None = None, exchange: str = "auto") -> _lib.Context:
    """Native context for this rank of an initialised torch.distributed job.

    ``exchange``: "nccl" (the library's NCCL communicator), "host" (torch.distributed
    all-reduce through a callback) or "auto" (NCCL when the group's backend is NCCL).
    With world size 1 this is a plain single-GPU context.  The context also
    becomes the process default, so ``boruvka_emst(points)`` on every rank
    computes one EMST cooperatively (all ranks must call it with the same points).
    """
    import torch.distributed as dist

    if device is None:
        device = int(os.environ.get("LOCAL_RANK", "0"))
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        ctx = _lib.Context(device)
    else:
        if exchange == "auto":
            exchange = "nccl" if dist.get_backend(group) == "nccl" else "host"
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        if exchange == "nccl":
            ctx = _lib.Context(device, rank, world, broadcast_nccl_id(group))
        elif exchange == "host":
            ctx = _lib.Context(device, rank, world, None)
            ctx.set_exchange(host_allreduce(group))
        else:
            raise ValueError(f"exchange must be 'nccl', 'host' or 'auto', got {exchange!r}")
        ctx.exchange = exchange
    _lib.set_default_context(ctx)
    return ctx
