"""The tree-level public API around the hot path, against goldens recorded from the reference
(tests/golden/make_goldens.py api): Bvh.sweep_order / sweep_starts (bvh.py:293-302), morton_codes /
sort_by_morton with caller bounds and morton_encode (geometry.py:209-254) on the GPU, and the host-side
callback walks traverse_nearest / for_each_leaf_to_root (bvh.py:343-440)."""

import json
import os

import numpy as np
import pytest

import paper_2207_00514_b200 as E

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def api():
    with open(os.path.join(GOLDEN, "api.json")) as fh:
        meta = json.load(fh)
    return np.load(os.path.join(GOLDEN, "api.npz")), meta["cases"]


def _tree(a, p):
    pts = a[p + "points"]
    return E.Bvh(pts.shape[0], pts.shape[1], a[p + "leaf_perm"], a[p + "left"], a[p + "right"], a[p + "parent"],
                 a[p + "leaf_parent"], a[p + "box_lo"], a[p + "box_hi"], a[p + "sweep_order"], a[p + "sweep_starts"])


def test_traverse_nearest_call_sequences(api):
    a, cases = api
    walked = 0
    for name in cases:
        p = name + "/"
        if p + "queries" not in a:
            continue
        pts, tree = a[p + "points"], _tree(a, p)
        for j, q in enumerate(a[p + "queries"]):
            seen = []

            def on_leaf(i, dist):
                seen.append((i, dist))
                return dist if dist > 0 else None

            r = E.traverse_nearest(tree, pts, q, on_leaf=on_leaf)
            assert [i for i, _ in seen] == a[p + f"walk{j}_pts"].tolist(), (name, j)
            assert np.array_equal(np.array([d for _, d in seen]), a[p + f"walk{j}_dist"]), (name, j)
            assert r == a[p + f"walk{j}_radius"][0]
            pruned, got = [], []

            def prune(ref, lb, radius):
                pruned.append((ref, lb))
                return lb > 0.25 * (1 + (ref % 3))

            E.traverse_nearest(tree, pts, q, on_leaf=lambda i, d: got.append(i), prune=prune, radius=0.5)
            assert [x for x, _ in pruned] == a[p + f"prune{j}_refs"].tolist(), (name, j)
            assert np.array_equal(np.array([b for _, b in pruned]), a[p + f"prune{j}_lbs"])
            assert got == a[p + f"prune{j}_pts"].tolist()
            walked += 1
    assert walked >= 12


def test_for_each_leaf_to_root_order(api):
    a, cases = api
    for name in cases:
        p = name + "/"
        if p + "sweep_visits" not in a:
            continue
        tree = _tree(a, p)
        order = []
        E.for_each_leaf_to_root(tree, order.append)
        assert order == a[p + "sweep_visits"].tolist()
        stop = []
        E.for_each_leaf_to_root(tree, lambda v: (stop.append(v), v % 5 != 0)[1])
        assert stop == a[p + "sweep_visits_stop"].tolist()


def test_traverse_nearest_errors(api):
    a, cases = api
    p = cases[0] + "/"
    tree = _tree(a, p)
    with pytest.raises(E.DimensionMismatchError):
        E.traverse_nearest(tree, a[p + "points"][:-1], a[p + "points"][0], on_leaf=lambda i, d: None)
    with pytest.raises(E.DimensionMismatchError):
        E.traverse_nearest(tree, a[p + "points"], np.zeros(5), on_leaf=lambda i, d: None)


def test_morton_encode_validation():
    b = E.Aabb(np.zeros(3), np.ones(3))
    with pytest.raises(E.UnsupportedDimensionError):
        E.morton_encode(np.zeros((2, 3)), b)
    with pytest.raises(E.DimensionMismatchError):
        E.morton_encode(np.zeros(2), b)
    with pytest.raises(E.InvalidCoordinateError):
        E.morton_encode(np.array([0.0, np.nan, 0.0]), b)


@pytest.mark.gpu
def test_level_schedule_matches_reference(api):
    a, cases = api
    for name in cases:
        p = name + "/"
        tree = E.build(a[p + "points"])
        assert np.array_equal(tree.sweep_order, a[p + "sweep_order"]), name
        assert np.array_equal(tree.sweep_starts, a[p + "sweep_starts"]), name


@pytest.mark.gpu
def test_morton_with_caller_bounds(api):
    a, cases = api
    for name in cases:
        p = name + "/"
        pts = a[p + "points"]
        for tag in ("inner", "outer", "flat"):
            lo, hi = a[p + f"bounds_{tag}"]
            b = E.Aabb(lo, hi)
            assert np.array_equal(E.morton_codes(pts, b), a[p + f"codes_{tag}"]), (name, tag)
            assert np.array_equal(E.sort_by_morton(pts, b), a[p + f"perm_{tag}"]), (name, tag)
            enc = [E.morton_encode(x, b) for x in pts[:16]]
            assert enc == a[p + f"encode_{tag}"].tolist(), (name, tag)
        # default bounds: the tight scene box, the build's own order
        assert np.array_equal(E.sort_by_morton(pts), a[p + "leaf_perm"]), name


@pytest.mark.gpu
def test_built_tree_walks_like_the_reference(api):
    """traverse_nearest over the GPU-built arrays gives the reference's call sequence."""
    a, cases = api
    p = "normal3d_1000_s1/"
    pts = a[p + "points"]
    tree = E.build(pts)
    for j, q in enumerate(a[p + "queries"]):
        seen = []
        E.traverse_nearest(tree, pts, q, on_leaf=lambda i, d: (seen.append(i), d if d > 0 else None)[1])
        assert seen == a[p + f"walk{j}_pts"].tolist()
