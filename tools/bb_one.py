import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2207_00514_b200 as E
pts = E.generate(E.DatasetSpec("normal", 10_000_000, 3, seed=0))
bvh = E.build(pts)
state = E.ComponentState.initial(bvh, device="cuda")
for r in range(7):
    E.reduce_labels(bvh, state)
    E.compute_upper_bounds(state, bvh.leaf_perm, pts)
    if r == 6: torch.cuda.cudart().cudaProfilerStart()
    out = E.find_component_outgoing_edges(bvh, pts, state)
    if r == 6: torch.cuda.synchronize(); torch.cuda.cudart().cudaProfilerStop()
    E.merge_components(state, out)
