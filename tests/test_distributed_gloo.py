"""World-size-2 CPU tests (gloo) of the multi-GPU host logic.

Covers what the N>1 path adds on top of the single-GPU kernels: the Morton
shard plan, the NCCL-id rendezvous over torch.distributed, and the exactness
of the two-phase min exchange (checked on oracle shards, since there is no GPU
here).  The native NCCL path itself runs in bench.py under torchrun.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

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
    w = torch.from_numpy(bw.copy()).view(torch.int64)
    uv = torch.from_numpy(np.where(bv >= 0, (bu << 32) | np.maximum(bv, 0), np.iinfo(np.int64).max))
    return w, uv


def _worker(rank, world, port, case, out):
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
        w_min, uv_min = D.exchange_component_minima(w, uv)
        nid = D.broadcast_nccl_id()
        if rank == 0:
            np.savez(out, w=w_min.numpy(), uv=uv_min.numpy(), nid=np.frombuffer(nid, np.uint8))
        else:
            np.savez(out + f".{rank}", nid=np.frombuffer(nid, np.uint8))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
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
        assert np.array_equal(w[reps], arrays[p + "best_w"])
        assert np.array_equal(got["uv"][reps] >> 32, arrays[p + "best_u"])
        assert np.array_equal(got["uv"][reps] & 0xFFFFFFFF, arrays[p + "best_v"])
        # every rank received rank 0's NCCL id
        other = np.load(out + ".1.npz")
        assert np.array_equal(other["nid"], got["nid"]) and got["nid"].size == 128
