"""Mutual reachability on the GPU against the reference's own outputs.

Goldens: tests/golden/mrd.{npz,json}, recorded by ``make_goldens.py mrd`` from the
reference (metric.py compute_core_distances; mst.py boruvka_emst(metric="mrd",
k_pts) and boruvka_emst(MutualReachability(CoreDistances))).  Bar: core
distances bit-equal, MST edges and weights bit-equal, equal iterations,
component counts and total weight (criteria 2 and 6 of the reference's
acceptance suite, test_acceptance.py:80-202).
"""

import numpy as np
import pytest

import paper_2207_00514_b200 as E

pytestmark = pytest.mark.gpu


def _keys(meta):
    return sorted(k for k in meta["cases"] if k != "given")


def test_core_distances_match_reference(mrd_golden):
    arrays, meta = mrd_golden
    for key in _keys(meta):
        name, k = key.rsplit("/", 1)
        pts = arrays[name + "/points"]
        got = E.compute_core_distances(E.build(pts), pts, int(k[1:])).values
        assert np.array_equal(got, arrays[key + "/core"]), key


def test_mrd_mst_matches_reference(mrd_golden):
    arrays, meta = mrd_golden
    for key in _keys(meta):
        name, k = key.rsplit("/", 1)
        rec = meta["cases"][key]
        res = E.boruvka_emst(arrays[name + "/points"], metric="mrd", k_pts=int(k[1:]))
        assert np.array_equal(res.edges, arrays[key + "/edges"]), key
        assert np.array_equal(res.weights, arrays[key + "/weights"]), key
        assert res.iterations == rec["iterations"], key
        assert res.component_counts == rec["component_counts"], key
        assert res.total_weight == rec["total_weight"], key
        assert res.phase_timings["core"] > 0.0, key


@pytest.mark.parametrize("skip,bounds", [(False, True), (True, False), (False, False)])
def test_mrd_flags_do_not_change_the_result(mrd_golden, skip, bounds):
    arrays, meta = mrd_golden
    for key in ("blobs3d_5000_s4/k4", "uniform2d_1000_s3/k16", "normal3d_5000_s4/k2"):
        name, k = key.rsplit("/", 1)
        res = E.boruvka_emst(arrays[name + "/points"], metric="mrd", k_pts=int(k[1:]), subtree_skip=skip,
                             upper_bound_seeding=bounds)
        assert np.array_equal(res.edges, arrays[key + "/edges"]), key
        assert np.array_equal(res.weights, arrays[key + "/weights"]), key


def test_given_core_table(mrd_golden):
    arrays, meta = mrd_golden
    core = E.CoreDistances(4, arrays["given/core"])
    res = E.boruvka_emst(arrays["given/points"], metric=E.MutualReachability(core))
    assert np.array_equal(res.edges, arrays["given/edges"])
    assert np.array_equal(res.weights, arrays["given/weights"])
    assert res.total_weight == meta["cases"]["given"]["total_weight"]


def test_k1_is_euclidean_bit_for_bit():
    for kind, d in (("uniform", 2), ("normal", 3), ("blobs", 3)):
        pts = E.generate(E.DatasetSpec(kind, 1000, d, seed=0))
        a = E.boruvka_emst(pts)
        b = E.boruvka_emst(pts, metric="mrd", k_pts=1)
        assert np.array_equal(a.edges, b.edges) and np.array_equal(a.weights, b.weights)


def test_mrd_virtual_shards_are_byte_identical(mrd_golden):
    arrays, meta = mrd_golden
    key = "blobs3d_20000_s5/k4"
    pts = arrays["blobs3d_20000_s5/points"]
    for shards in (2, 3):
        ctx = E.Context(0)
        ctx.set_virtual_shards(shards)
        res = E.boruvka_emst(pts, metric="mrd", k_pts=4, context=ctx)
        assert np.array_equal(res.edges, arrays[key + "/edges"]), shards
        assert np.array_equal(res.weights, arrays[key + "/weights"]), shards


def test_mrd_parameter_errors():
    pts = E.generate(E.DatasetSpec("uniform", 10, 3, seed=0))
    with pytest.raises(E.InvalidParameterError):
        E.boruvka_emst(pts, metric="mrd", k_pts=11)   # k_pts > n
    with pytest.raises(E.InvalidParameterError):
        E.compute_core_distances(E.build(pts), pts, 0)
    with pytest.raises(E.DimensionMismatchError):
        E.boruvka_emst(pts, metric=E.MutualReachability(E.CoreDistances(2, np.zeros(9))))
    assert np.array_equal(E.compute_core_distances(E.build(pts), pts, 1).values, np.zeros(10))


def test_mrd_building_blocks(mrd_golden):
    """compute_upper_bounds / find_component_outgoing_edges under a MutualReachability metric."""
    arrays, meta = mrd_golden
    pts = arrays["normal3d_1000_s3/points"]
    core = arrays["normal3d_1000_s3/k4/core"]
    metric = E.MutualReachability(E.CoreDistances(4, core))
    tree = E.build(pts)
    n = len(pts)
    state = E.ComponentState(np.arange(n, dtype=np.int64), np.full(n - 1, E.MIXED, np.int64), np.full(n, np.inf))
    ub = E.compute_upper_bounds(state, tree.leaf_perm, pts, metric).copy()
    p64 = pts.astype(np.float64)
    perm = np.asarray(tree.leaf_perm)
    want = np.full(n, np.inf)
    for s in range(n - 1):
        a, b = perm[s], perm[s + 1]
        w = max(float(np.sqrt(((p64[a] - p64[b]) ** 2).sum())), core[a], core[b])
        want[a] = min(want[a], w)
        want[b] = min(want[b], w)
    assert np.array_equal(ub, want)
    out = E.find_component_outgoing_edges(tree, pts, state, metric)
    # round 1 with singletons: each point's best edge is its mutual-reachability nearest neighbour
    assert np.isfinite(out.w[out.reps]).all() and out.w[out.reps].min() == arrays["normal3d_1000_s3/k4/weights"][0]


def test_run_bench_reports():
    """run_bench: the reference's report rows, on the GPU path."""
    pts = E.generate(E.DatasetSpec("blobs", 20_000, 3, seed=0))
    reps = E.run_bench(pts, [5_000, 20_000], repeats=2, dataset="blobs")
    assert [r.n for r in reps] == [5_000, 20_000]
    assert all(r.rate > 0 and r.t_total >= r.t_tree and r.iterations > 0 for r in reps)
    assert np.isnan(reps[0].time_ratio_prev) and reps[1].time_ratio_prev > 0
    assert reps[0].row().count("\t") == E.BenchReport.HEADER.count("\t")
    mrd = E.run_bench(pts, [10_000], repeats=1, metric="mrd", k_pts=4)
    assert mrd[0].t_core > 0
