"""Pin the CPU oracle (oracle/emst_oracle.c) against golden vectors from the reference.

The goldens were recorded by running the reference package itself
(tests/golden/make_goldens.py).  Everything here is CPU-only.
"""

import numpy as np
import pytest

from _golden import array_digest, digest
from oracle import oracle as orc
from paper_2207_00514_b200.data import DatasetSpec, generate


def _case_names(meta):
    return sorted(meta["cases"].keys())


def test_generator_matches_reference_bytes(small_golden):
    _, meta = small_golden
    for name, rec in meta["cases"].items():
        if "spec" not in rec:
            continue
        s = rec["spec"]
        kw = {k: s[k] for k in ("blobs", "spread") if k in s}
        pts = generate(DatasetSpec(s["kind"], s["n"], s["d"], s["seed"], **kw))
        assert array_digest(pts) == rec["points_digest"], name
    for key, rec in list(meta["matrix"].items())[::7]:
        kind, d, n, seed = key.split("_")
        pts = generate(DatasetSpec(kind, int(n), int(d[0]), int(seed[1:])))
        assert array_digest(pts) == rec["points_digest"], key


@pytest.mark.parametrize("which", ["codes", "build"])
def test_oracle_build_arrays(small_golden, which):
    arrays, meta = small_golden
    for name in _case_names(meta):
        pts = arrays[name + "/points"]
        if which == "codes":
            assert np.array_equal(orc.morton_codes(pts), arrays[name + "/codes"]), name
            continue
        t = orc.build_tree(pts)
        for field in ("perm", "left", "right", "parent", "leaf_parent"):
            want = arrays[name + "/" + field]
            assert np.array_equal(getattr(t, field), want), (name, field)
        assert np.array_equal(t.box_lo, arrays[name + "/box_lo"]), name
        assert np.array_equal(t.box_hi, arrays[name + "/box_hi"]), name


def test_oracle_mst_cases(small_golden):
    arrays, meta = small_golden
    for name in _case_names(meta):
        rec = meta["cases"][name]
        pts = arrays[name + "/points"]
        res = orc.boruvka_emst(pts)
        assert np.array_equal(res.edges, arrays[name + "/edges"]), name
        assert np.array_equal(res.weights, arrays[name + "/weights"]), name
        assert res.iterations == rec["iterations"], name
        assert res.component_counts == rec["component_counts"], name
        assert res.total_weight == rec["total_weight"], name
        # identical traversal order => identical work counter
        assert res.leaf_distance_evals == rec["leaf_distance_evals"], name
        noopt = orc.boruvka_emst(pts, subtree_skip=False, upper_bound_seeding=False)
        assert noopt.leaf_distance_evals == rec["leaf_distance_evals_noopt"], name
        assert np.array_equal(noopt.edges, res.edges)


def test_oracle_rounds(small_golden):
    """Per-round building blocks vs the reference's (mst.py:436-547)."""
    arrays, meta = small_golden
    for name in _case_names(meta):
        rec = meta["cases"][name]
        pts = arrays[name + "/points"]
        perm = arrays[name + "/perm"]
        for k in range(rec.get("rounds", 0)):
            p = f"{name}/r{k}_"
            labels = arrays[p + "labels_in"]
            il = orc.reduce_labels(pts, labels)
            assert np.array_equal(il, arrays[p + "internal_labels"]), (name, k)
            ub = orc.upper_bounds(pts, perm, labels)
            assert np.array_equal(ub, arrays[p + "upper_bounds"]), (name, k)
            bu, bv, bw, _ = orc.find_edges(pts, labels, il, ub)
            reps = arrays[p + "reps"]
            assert np.array_equal(bu[reps], arrays[p + "best_u"]), (name, k)
            assert np.array_equal(bv[reps], arrays[p + "best_v"]), (name, k)
            assert np.array_equal(bw[reps], arrays[p + "best_w"]), (name, k)
            lab, eu, ev, ew, nr = orc.merge(labels, reps, bu, bv, bw)
            assert np.array_equal(eu, arrays[p + "edge_u"]), (name, k)
            assert np.array_equal(ev, arrays[p + "edge_v"]), (name, k)
            assert np.array_equal(ew, arrays[p + "edge_w"]), (name, k)
            assert np.array_equal(nr, arrays[p + "new_reps"]), (name, k)
            assert np.array_equal(lab, arrays[p + "labels_out"]), (name, k)


def test_oracle_sharded_find_edges_combines_to_global(small_golden):
    """Sharding queries by Morton slot range and min-combining is exact."""
    arrays, meta = small_golden
    name = "blobs3d_3000_s2"
    pts = arrays[name + "/points"]
    labels = arrays[name + "/r1_labels_in"]
    il = arrays[name + "/r1_internal_labels"]
    ub = arrays[name + "/r1_upper_bounds"]
    reps = arrays[name + "/r1_reps"]
    n = pts.shape[0]
    full = orc.find_edges(pts, labels, il, ub)
    for p in (2, 3, 8):
        cuts = [g * n // p for g in range(p + 1)]
        parts = [orc.find_edges(pts, labels, il, ub, q_begin=cuts[g], q_end=cuts[g + 1]) for g in range(p)]
        w = np.min([pp[2] for pp in parts], axis=0)
        uv = np.full(n, np.iinfo(np.int64).max)
        for pp in parts:
            cand = np.where(pp[2] == w, (pp[0] << 32) | np.maximum(pp[1], 0), np.iinfo(np.int64).max)
            uv = np.minimum(uv, cand)
        assert np.array_equal(w[reps], full[2][reps])
        assert np.array_equal(uv[reps] >> 32, full[0][reps])
        assert np.array_equal(uv[reps] & 0xFFFFFFFF, full[1][reps])


def test_oracle_acceptance_matrix(small_golden):
    """SPEC criterion 1 matrix (test_acceptance.py:54-78): 180 digests."""
    _, meta = small_golden
    for key, rec in meta["matrix"].items():
        kind, d, n, seed = key.split("_")
        pts = generate(DatasetSpec(kind, int(n), int(d[0]), int(seed[1:])))
        res = orc.boruvka_emst(pts)
        assert digest(res.edges, res.weights) == rec["digest"], key
        assert res.iterations == rec["iterations"], key
        assert res.component_counts == rec["component_counts"], key


@pytest.mark.parametrize("name", ["uniform3d_100k", "uniform3d_1m", "blobs3d_1m", "blobs2d_1m", "normal3d_1m"])
def test_oracle_large(large_golden, name):
    if name not in large_golden:
        pytest.skip(f"{name} not recorded")
    rec = large_golden[name]
    s = rec["spec"]
    pts = generate(DatasetSpec(s["kind"], s["n"], s["d"], s["seed"]))
    assert array_digest(pts) == rec["points_digest"]
    res = orc.boruvka_emst(pts)
    assert digest(res.edges, res.weights) == rec["digest"]
    assert res.iterations == rec["iterations"]
    assert res.component_counts == rec["component_counts"]
    assert res.total_weight == rec["total_weight"]
    assert res.leaf_distance_evals == rec["leaf_distance_evals"]


# ---------------------------------------------------------------- mutual reachability (§8f row 1)

def test_oracle_core_distances_match_reference(mrd_golden):
    """metric.py compute_core_distances, restated in oracle/emst_oracle.c, against the reference's values."""
    arrays, meta = mrd_golden
    for key in sorted(k for k in meta["cases"] if k != "given"):
        name, k = key.rsplit("/", 1)
        got = orc.core_distances(arrays[name + "/points"], int(k[1:]))
        assert np.array_equal(got, arrays[key + "/core"]), key


def test_oracle_mrd_mst_matches_reference(mrd_golden):
    arrays, meta = mrd_golden
    for key in sorted(k for k in meta["cases"] if k != "given"):
        name, k = key.rsplit("/", 1)
        rec = meta["cases"][key]
        res = orc.boruvka_emst(arrays[name + "/points"], k_pts=int(k[1:]))
        assert np.array_equal(res.edges, arrays[key + "/edges"]), key
        assert np.array_equal(res.weights, arrays[key + "/weights"]), key
        assert res.iterations == rec["iterations"] and res.component_counts == rec["component_counts"], key
        assert res.total_weight == rec["total_weight"], key
    res = orc.boruvka_emst(arrays["given/points"], cores=arrays["given/core"])
    assert np.array_equal(res.edges, arrays["given/edges"]) and np.array_equal(res.weights, arrays["given/weights"])
