import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2207_00514_b200 as E
pts = E.generate(E.DatasetSpec("normal", 10_000_000, 3, seed=0))
bvh = E.build(pts)
for dev in ("cuda", "cuda", "cuda"):
    state = E.ComponentState.initial(bvh, device=dev)
    T = {"nc":0, "rl":0, "ub":0, "find":0, "merge":0}
    t00 = time.perf_counter()
    while True:
        torch.cuda.synchronize(); t = time.perf_counter(); k = state.num_components; T["nc"] += time.perf_counter()-t
        if k <= 1: break
        t = time.perf_counter(); E.reduce_labels(bvh, state); T["rl"] += time.perf_counter()-t
        t = time.perf_counter(); E.compute_upper_bounds(state, bvh.leaf_perm, pts); T["ub"] += time.perf_counter()-t
        t = time.perf_counter(); out = E.find_component_outgoing_edges(bvh, pts, state); T["find"] += time.perf_counter()-t
        t = time.perf_counter(); E.merge_components(state, out); T["merge"] += time.perf_counter()-t
    print(dev, "total", round((time.perf_counter()-t00)*1e3,1), {k: round(v*1e3,1) for k,v in T.items()})
