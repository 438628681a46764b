"""Mutual-reachability timing at scale (developer tool): python tools/mrd_timing.py [cfg] [k]."""
import sys, time
import numpy as np, torch
import paper_2207_00514_b200 as E

cfg = sys.argv[1] if len(sys.argv) > 1 else "blobs3d_37m"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
kind, rest = cfg[:-6], cfg
specs = {"blobs3d_37m": ("blobs", 37_000_000, 3), "blobs2d_24m": ("blobs", 24_000_000, 2),
         "uniform3d_1m": ("uniform", 1_000_000, 3), "blobs3d_1m": ("blobs", 1_000_000, 3)}
kind, n, d = specs[cfg]
pts = E.generate(E.DatasetSpec(kind, n, d, seed=0))
pinned = torch.from_numpy(pts).pin_memory().numpy()
ctx = E.Context(0)
for it in range(3):
    t0 = time.perf_counter()
    res = E.boruvka_emst(pinned, metric="mrd", k_pts=k, context=ctx)
    dt = time.perf_counter() - t0
    t = res.phase_timings
    print(f"{cfg} k={k}: {dt*1e3:.1f} ms e2e  tree {t['tree']*1e3:.1f} core {t['core']*1e3:.1f} "
          f"find {t['find_edges']*1e3:.1f} mst {t['mst']*1e3:.1f} iters {res.iterations} W={res.total_weight!r}")
