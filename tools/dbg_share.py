import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2207_00514_b200 as E
from oracle import oracle as orc
g = np.arange(40, dtype=np.float32) / 4
lattice = np.stack(np.meshgrid(g, g, indexing="ij"), -1).reshape(-1, 2)
clouds = {"blobs3": E.generate(E.DatasetSpec("blobs", 60_000, 3, seed=3)),
          "uni2": E.generate(E.DatasetSpec("uniform", 60_000, 2, seed=4)),
          "norm3": E.generate(E.DatasetSpec("normal", 60_000, 3, seed=5)), "lattice": lattice}
for name, pts in clouds.items():
    try:
        got = E.boruvka_emst(pts)
        ref = orc.boruvka_emst(pts)
        print(name, "ok" if np.array_equal(got.edges, ref.edges) else "DIFF", got.iterations)
    except Exception as e:
        print(name, "FAIL", e)
    # per round through the building blocks vs oracle
    bvh = E.build(pts)
    state = E.ComponentState.initial(bvh)
    r = 0
    while state.num_components > 1 and r < 30:
        r += 1
        E.reduce_labels(bvh, state)
        E.compute_upper_bounds(state, bvh.leaf_perm, pts)
        out = E.find_component_outgoing_edges(bvh, pts, state)
        il = orc.reduce_labels(pts, state.labels)
        ub = orc.upper_bounds(pts, orc.sort_by_morton(pts), state.labels)
        ou, ov, ow = orc.find_edges(pts, state.labels, il, ub)[:3]
        reps = out.reps
        bad = reps[(out.w[reps] != ow[reps]) | (out.v[reps] != ov[reps])]
        if len(bad):
            k = bad[0]
            print(f"  round {r}: {len(bad)} of {len(reps)} comps differ; e.g. rep {k}: gpu ({out.u[k]},{out.v[k]},{out.w[k]!r}) oracle ({ou[k]},{ov[k]},{ow[k]!r}) size {np.count_nonzero(state.labels==k)}")
            break
        E.merge_components(state, out)
