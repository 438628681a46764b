"""Per-call times of the device building-block loop vs the solve (developer tool; EMST_TRACE=1 for traversal lines)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2207_00514_b200 as E
pts = E.generate(E.DatasetSpec("normal", 10_000_000, 3, seed=0))
bvh = E.build(pts)
for rep in range(2):
    state = E.ComponentState.initial(bvh, device="cuda")
    r = 0
    while state.num_components > 1:
        r += 1
        E.reduce_labels(bvh, state)
        E.compute_upper_bounds(state, bvh.leaf_perm, pts)
        torch.cuda.synchronize(); t = time.perf_counter()
        out = E.find_component_outgoing_edges(bvh, pts, state)
        torch.cuda.synchronize(); tf = time.perf_counter() - t
        E.merge_components(state, out)
        if rep: print(f"round {r}: find {tf * 1e3:.2f} ms evals {out.leaf_distance_evals}", file=sys.stderr, flush=True)
res = E.boruvka_emst(pts)
print("solve", res.phase_timings, file=sys.stderr)
