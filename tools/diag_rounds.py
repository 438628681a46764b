"""Developer diagnostic: locate the first per-round divergence between the GPU path and the oracle."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2207_00514_b200 as E
from oracle import oracle as orc


def check(kind, n, d, seed, **kw):
    pts = E.generate(E.DatasetSpec(kind, n, d, seed, **kw))
    want = orc.boruvka_emst(pts)
    runs = [E.boruvka_emst(pts) for _ in range(3)]
    same = all(np.array_equal(r.edges, runs[0].edges) for r in runs)
    ok = np.array_equal(runs[0].edges, want.edges) and np.array_equal(runs[0].weights, want.weights)
    print(f"{kind} {d}D n={n} s={seed}: ok={ok} deterministic={same} gpu_counts={runs[0].component_counts} "
          f"ref_counts={want.component_counts}")
    if ok:
        return
    for flags in [(True, True), (False, True), (True, False), (False, False)]:
        r = E.boruvka_emst(pts, subtree_skip=flags[0], upper_bound_seeding=flags[1])
        print("  flags", flags, "ok", np.array_equal(r.edges, want.edges))
    # per-round building blocks along the oracle's trajectory
    tree = E.build(pts)
    otree = orc.build_tree(pts)
    print("  tree equal:", np.array_equal(tree.leaf_perm, otree.perm), np.array_equal(tree.left, otree.left),
          np.array_equal(tree.box_lo, otree.box_lo))
    labels = np.arange(n, dtype=np.int64)
    for k in range(40):
        reps = np.unique(labels)
        if len(reps) < 2:
            break
        il = orc.reduce_labels(pts, labels)
        ub = orc.upper_bounds(pts, otree.perm, labels)
        st = E.ComponentState(labels.copy(), np.full(n - 1, -1, np.int64), np.full(n, np.inf))
        gil = E.reduce_labels(tree, st)
        gub = E.compute_upper_bounds(st, tree.leaf_perm, pts)
        print(f"  round {k}: comps={len(reps)} il_eq={np.array_equal(gil, il)} ub_eq={np.array_equal(gub, ub)}")
        bu, bv, bw, _ = orc.find_edges(pts, labels, il, ub)
        st.upper_bounds[:] = ub
        out = E.find_component_outgoing_edges(tree, pts, st)
        bad = reps[(out.u[reps] != bu[reps]) | (out.v[reps] != bv[reps]) | (out.w[reps] != bw[reps])]
        print(f"    find mismatches: {len(bad)}")
        for r in bad[:5]:
            print(f"      rep {r}: gpu ({out.u[r]},{out.v[r]},{out.w[r]!r}) ref ({bu[r]},{bv[r]},{bw[r]!r}) ub={ub[r]!r}")
        lab, eu, ev, ew, nr = orc.merge(labels, reps, bu, bv, bw)
        st2 = E.ComponentState(labels.copy(), np.full(n - 1, -1, np.int64), np.full(n, np.inf))
        o2 = E.OutgoingEdges(reps, bu, bv, bw, 0)
        res = E.merge_components(st2, o2)
        print(f"    merge eq: labels={np.array_equal(st2.labels, lab)} edges={np.array_equal(res.edge_u, eu)} "
              f"new_reps={np.array_equal(res.new_reps, nr)}")
        labels = lab


if __name__ == "__main__":
    check("uniform", 2000, 3, 0)
    check("blobs", 20000, 3, 0)
    check("uniform", 1000, 3, 0)
    check("uniform", 2000, 2, 0)
