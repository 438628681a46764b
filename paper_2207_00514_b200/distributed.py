"""Multi-GPU plumbing: one process per GPU, torch.distributed for the rendezvous.

The tree is replicated (every rank builds the same one from the same points,
deterministically), each Boruvka round's traversal is split by Morton slot
range, and the per-component minima meet in a two-phase NCCL min-allreduce
issued by the native library on its own communicator:

  phase A  allreduce-min of the f64 weight bit patterns, one u64 per component;
  phase B  allreduce-min of (u << 32 | v) over the ranks whose local weight
           equals the global one (all-ones elsewhere).

u64 min on the bit pattern of a non-negative double is the numeric min, and
phase B then picks the smallest (u, v) among the minimum-weight candidates, so
the pair of u64 reductions is exactly the reference's 128-bit (w, u, v) order
(mst.py:62-89) -- a single u64 allreduce of a truncated key would not be.

torch.distributed only carries the 128-byte NCCL unique id from rank 0 to the
others; the per-round collectives run inside ``libemst_b200.so``.
"""

from __future__ import annotations

import os

from . import _lib


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Morton slot range [begin, end) of `rank`'s queries (same formula as the C++ side)."""
    return rank * n // world, (rank + 1) * n // world


def broadcast_nccl_id(group=None) -> bytes:
    """Create the NCCL unique id on rank 0 and hand it to every rank of `group`."""
    import torch.distributed as dist

    obj = [_lib.nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return obj[0]


def init_context(group=None, device: int | None = None) -> _lib.Context:
    """Native context for this rank of an initialised torch.distributed job.

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
        nid = broadcast_nccl_id(group)
        ctx = _lib.Context(device, dist.get_rank(group), dist.get_world_size(group), nid)
    _lib.set_default_context(ctx)
    return ctx


def exchange_component_minima(w_bits, uv, group=None):
    """The two-phase exchange on torch tensors (int64 views of the u64 keys).

    Mirrors k_split_keys / ncclAllReduce / k_mask_uv / ncclAllReduce / k_join_keys
    in csrc/emst_b200.cu; works with any backend (the CPU tests run it on gloo).
    Keys are non-negative as int64: w >= 0 has a clear sign bit and u, v < 2^31.
    """
    import torch
    import torch.distributed as dist

    w_min = w_bits.clone()
    dist.all_reduce(w_min, op=dist.ReduceOp.MIN, group=group)
    none = torch.iinfo(torch.int64).max
    masked = torch.where(w_bits == w_min, uv, torch.full_like(uv, none))
    dist.all_reduce(masked, op=dist.ReduceOp.MIN, group=group)
    return w_min, masked
