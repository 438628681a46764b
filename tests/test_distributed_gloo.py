"""World-size-2/3 CPU tests (gloo) of the multi-GPU host logic.

Covers what the N>1 path adds on top of the single-GPU kernels: the Morton
shard plan, the NCCL-id rendezvous over torch.distributed, and the exactness
of the two-phase min exchange through the host all-reduce the library calls
back into (distributed.host_allreduce, checked on oracle shards since there is
no GPU here).  tests/test_gpu_multirank.py runs the native path itself: N
processes, each with its own context, sharding the traversal on one GPU.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2207_00514_b200 as E
from paper_2207_00514_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_shard_ranges_partition_slots():
    for n in (1, 2, 7, 1000, 37_000_000):
        for world in (1, 2, 3, 4, 8):
            cuts = [D.shard_range(n, r, world) for r in range(world)]
            assert cuts[0][0] == 0 and cuts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(cuts, cuts[1:]))
            assert all(e - b in (n // world, n // world + 1) for b, e in cuts)


def _keys(bu, bv, bw):
    """The device's EdgeKey halves: f64 weight bits, u << 32 | v; all-ones where none (k_split_keys' input)."""
    w = np.where(bv >= 0, bw.view(np.uint64), np.uint64(~np.uint64(0)))
    uv = np.where(bv >= 0, (bu.astype(np.uint64) << np.uint64(32)) | np.maximum(bv, 0).astype(np.uint64),
                  np.uint64(~np.uint64(0)))
    return w.astype(np.uint64), uv.astype(np.uint64)


def _worker(rank, world, port, case, out):
    """One rank: oracle keys of its Morton shard, then the two-phase exchange through the host all-reduce
    the native library calls back into (distributed.host_allreduce), with the split / mask / join steps of
    csrc/boruvka.cuh restated in numpy."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as orc
        pts, labels, il, ub = (np.load(case)[k] for k in ("pts", "labels", "il", "ub"))
        n = pts.shape[0]
        b, e = D.shard_range(n, rank, world)
        bu, bv, bw, _ = orc.find_edges(pts, labels, il, ub, q_begin=b, q_end=e)
        w, uv = _keys(bu, bv, bw)
        allreduce = D.host_allreduce()
        xw = w.copy()                                        # k_split_keys
        allreduce(xw, E._lib.EXCHANGE_MIN)                   # phase A
        xuv = np.where(w == xw, uv, np.uint64(~np.uint64(0)))  # k_mask_uv
        allreduce(xuv, E._lib.EXCHANGE_MIN)                  # phase B
        total = np.array([np.uint64(rank + 1)], np.uint64)
        allreduce(total, E._lib.EXCHANGE_SUM)
        nid = D.broadcast_nccl_id()
        if rank == 0:
            np.savez(out, w=xw, uv=xuv, total=total, nid=np.frombuffer(nid, np.uint8))
        else:
            np.savez(out + f".{rank}", nid=np.frombuffer(nid, np.uint8))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_two_phase_exchange_is_exact_over_gloo(small_golden, tmp_path, world):
    arrays, _ = small_golden
    name = "blobs2d_tie_20000"   # 2D lattice-like data: many exact weight ties
    for rnd in (0, 1, 2):
        p = f"{name}/r{rnd}_"
        case = str(tmp_path / f"case{rnd}.npz")
        np.savez(case, pts=arrays[name + "/points"], labels=arrays[p + "labels_in"],
                 il=arrays[p + "internal_labels"], ub=arrays[p + "upper_bounds"])
        out = str(tmp_path / f"out{rnd}.npz")
        mp.spawn(_worker, args=(world, _free_port(), case, out), nprocs=world, join=True)
        got = np.load(out)
        reps = arrays[p + "reps"]
        w = got["w"].view(np.float64)
        assert int(got["total"][0]) == world * (world + 1) // 2
        assert np.array_equal(w[reps], arrays[p + "best_w"])
        assert np.array_equal(got["uv"][reps] >> 32, arrays[p + "best_u"])
        assert np.array_equal(got["uv"][reps] & 0xFFFFFFFF, arrays[p + "best_v"])
        # every rank received rank 0's NCCL id
        other = np.load(out + ".1.npz")
        assert np.array_equal(other["nid"], got["nid"]) and got["nid"].size == 128
