"""Morton-range shard balance of the traversal (developer tool).

Runs one solve with p virtual shards on one GPU (EMST_TRACE=1 prints every
shard's traversal time) and reports, per round, max / mean shard time: the
factor by which the slowest rank of a p-GPU run would trail the mean.
usage: EMST_TRACE=1 python tools/shard_balance.py blobs3d_37m 8 2> trace.txt; python tools/shard_balance.py --parse trace.txt
"""
import re
import sys
import os
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def parse(path):
    per = defaultdict(list)
    fronts = {}
    for line in open(path):
        m = re.search(r"round (\d+) traverse \[(\d+), (\d+)\): ([\d.]+) ms", line)
        if m:
            per[int(m.group(1))].append(float(m.group(4)))
        m = re.search(r"comps (\d+): (\d+) nodes still mixed", line)
        if m:
            fronts[len(fronts) + 2] = (int(m.group(1)), int(m.group(2)))   # (labels run from round 2 on)
    tot_max = tot_mean = 0.0
    for r in sorted(per):
        t = per[r]
        mx, mean = max(t), sum(t) / len(t)
        tot_max += mx
        tot_mean += mean
        fr = fronts.get(r)
        print(f"round {r:2d}: shards {len(t)}  mean {mean:7.3f} ms  max {mx:7.3f} ms  max/mean {mx / mean:5.2f}"
              + (f"  | comps {fr[0]}, mixed nodes {fr[1]}" if fr else ""))
    if per:
        print(f"all rounds: sum of max {tot_max:.3f} ms, sum of mean {tot_mean:.3f} ms, ratio {tot_max / tot_mean:.2f}")


def run(cfg, p):
    import bench
    import paper_2207_00514_b200 as E
    import torch
    kind, n, d, seed = bench.CONFIGS[cfg]
    pts = torch.from_numpy(E.generate(E.DatasetSpec(kind, n, d, seed=seed))).cuda()
    ctx = E._lib.Context(0)
    ctx.set_virtual_shards(p)
    E.boruvka_emst(pts, context=ctx)   # warm-up
    print("----- timed", file=sys.stderr, flush=True)
    E.boruvka_emst(pts, context=ctx)


if __name__ == "__main__":
    if sys.argv[1] == "--parse":
        parse(sys.argv[2])
    else:
        run(sys.argv[1], int(sys.argv[2]))
