"""Small solves for compute-sanitizer (developer tool): every kernel family of the path at smoke size.

  compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} python tools/sanitize.py

Runs Euclidean 3D / 2D solves (all optimisation-flag combinations), virtual shards (the two-phase
exchange on a 1-rank NCCL communicator), mutual reachability and the per-round building blocks,
each checked against the CPU oracle so a run that corrupts memory also fails loudly.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2207_00514_b200 as E  # noqa: E402
from oracle import oracle as orc  # noqa: E402

n3 = int(os.environ.get("SAN_N", "6000"))
cases = [("blobs", n3, 3), ("uniform", n3 // 2, 2), ("normal", 3000, 3)]
for kind, n, d in cases:
    pts = E.generate(E.DatasetSpec(kind, n, d, seed=1))
    want = orc.boruvka_emst(pts)
    for skip in (True, False):
        for ub in (True, False):
            got = E.boruvka_emst(pts, subtree_skip=skip, upper_bound_seeding=ub)
            assert np.array_equal(got.edges, want.edges) and np.array_equal(got.weights, want.weights), (kind, d, skip, ub)
    got = E.boruvka_emst(torch.from_numpy(pts).cuda())
    assert np.array_equal(got.edges, want.edges)
    ctx = E.Context(0)
    ctx.set_virtual_shards(3)
    got = E.boruvka_emst(pts, context=ctx)
    assert np.array_equal(got.edges, want.edges), "virtual shards"
    print(f"ok {kind} {d}D n={n}", flush=True)
pts = E.generate(E.DatasetSpec("blobs", 3000, 3, seed=2))
got = E.boruvka_emst(pts, "mrd", 4)
want = orc.boruvka_emst(pts, k_pts=4)
assert np.array_equal(got.edges, want.edges) and np.array_equal(got.weights, want.weights), "mrd"
# ties: coincident points and a grid
grid = np.stack(np.meshgrid(np.arange(40), np.arange(40)), -1).reshape(-1, 2).astype(np.float32)
got = E.boruvka_emst(grid)
want = orc.boruvka_emst(grid)
assert np.array_equal(got.edges, want.edges) and np.array_equal(got.weights, want.weights), "grid ties"
# per-round building blocks: a whole solve driven round by round from the host
pts = E.generate(E.DatasetSpec("blobs", 2000, 3, seed=3))
bvh = E.build(pts)
state = E.ComponentState.initial(bvh)
edges = 0
while state.num_components > 1:
    E.reduce_labels(bvh, state)
    E.compute_upper_bounds(state, bvh.leaf_perm, pts)
    out = E.find_component_outgoing_edges(bvh, pts, state)
    res = E.merge_components(state, out)
    edges += res.edges_u.shape[0] if hasattr(res, "edges_u") else 0
# the same loop on device-resident state (tree reuse, GPU merge, kept proofs)
state = E.ComponentState.initial(bvh, device="cuda")
while state.num_components > 1:
    E.reduce_labels(bvh, state)
    E.compute_upper_bounds(state, bvh.leaf_perm, pts)
    out = E.find_component_outgoing_edges(bvh, pts, state)
    res = E.merge_components(state, out)
print("ok mrd, ties, building blocks (host and device state)", flush=True)
print("SANITIZE DONE", flush=True)
