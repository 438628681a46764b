"""Record golden vectors from the reference package (run in the build container only).

This script imports the unmodified reference implementation from
``/root/reference/pkg/src`` (the ``emst`` package, numba-JIT CPU code) and records
its outputs so that the oracle restatement under ``oracle/`` and the CUDA product
can be pinned against the reference on machines where the reference is absent
(the GPU box never sees ``/root/reference``).

Usage (needs a writable numba cache because the reference tree is read-only)::

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_goldens.py small
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_goldens.py large

``small`` writes ``tests/golden/small.npz`` + ``tests/golden/small.json`` (seconds);
``mrd`` writes ``tests/golden/mrd.npz`` + ``tests/golden/mrd.json``: the mutual-reachability
metric (core distances for k_pts and the MSTs; reference metric.py / mst.py:638-644);
``api`` writes ``tests/golden/api.npz`` + ``api.json``: the tree-level API (level schedule, Morton codes
with caller bounds, traverse_nearest / for_each_leaf_to_root call sequences);
``large`` appends the full-size configurations of BASELINE.json to
``tests/golden/large.json`` (minutes: 10M-37M points on the host CPU).

Digest convention (same as SURVEY.md §8c): ``sha256(edges.tobytes() +
weights.tobytes()).hexdigest()[:16]`` over the reference's int64 (n-1, 2) edge
array and float64 weights, both C-contiguous little-endian.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _import_reference():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import emst  # noqa: E402  (reference package, read-only)
    return emst


def digest(edges, weights) -> str:
    e = np.ascontiguousarray(edges, dtype="<i8")
    w = np.ascontiguousarray(weights, dtype="<f8")
    return hashlib.sha256(e.tobytes() + w.tobytes()).hexdigest()[:16]


def array_digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def _mst_record(res) -> dict:
    return {
        "digest": digest(res.edges, res.weights),
        "iterations": int(res.iterations),
        "total_weight": float(res.total_weight),
        "component_counts": [int(c) for c in res.component_counts],
        "leaf_distance_evals": int(res.leaf_distance_evals),
    }


def _tie_inputs():
    """Hand-made tie/degenerate inputs mirrored from the reference tests."""
    cases = {}
    # unit square (test_oracle.py:43-49)
    cases["unit_square"] = np.float32([[0, 0], [1, 0], [0, 1], [1, 1]])
    # collinear ties (test_mst.py:165-177)
    cases["collinear4"] = np.float32([[0, 0], [1, 0], [2, 0], [3, 0]])
    # two points (test_mst.py:154-162)
    cases["two_points"] = np.float32([[0.0, 0.0], [3.0, 4.0]])
    # 9x9 and 20x20 grids (test_oracle.py:68-76, demos/04_verify_against_oracles.py:44-51)
    g9 = np.stack(np.meshgrid(np.arange(9), np.arange(9), indexing="ij"), -1)
    cases["grid9"] = g9.reshape(-1, 2).astype(np.float32)
    g20 = np.stack(np.meshgrid(np.arange(20), np.arange(20), indexing="ij"), -1)
    cases["grid20"] = g20.reshape(-1, 2).astype(np.float32)
    g3 = np.stack(np.meshgrid(np.arange(7), np.arange(6), np.arange(5), indexing="ij"), -1)
    cases["grid3d_7x6x5"] = g3.reshape(-1, 3).astype(np.float32)
    # coincident points (test_mst.py:378-394, test_acceptance.py:247-265)
    cases["coincident50_3d"] = np.zeros((50, 3), np.float32)
    cases["coincident50_2d"] = np.zeros((50, 2), np.float32)
    # 33 identical points plus a few others (test_bvh.py:131-139 flavour)
    rng = np.random.default_rng(7)
    dup = np.concatenate([np.tile(np.float32([[0.25, 0.75, 0.5]]), (33, 1)),
                          rng.random((17, 3)).astype(np.float32)])
    cases["dup33_3d"] = dup
    # code-tie stability (test_geometry.py:198-203)
    cases["codetie_2d"] = np.concatenate([np.tile(np.float32([[0.25, 0.75]]), (6, 1)),
                                          np.float32([[0.9, 0.9], [0.1, 0.1]])])
    # zero-extent axis (test_geometry.py:206-211)
    cases["zero_extent_2d"] = np.float32([[0.5, 1.0], [0.5, 2.0], [0.5, 3.0]])
    # integer lattice with heavy duplicate weights, 3D
    cases["lattice_dups_3d"] = rng.integers(0, 6, (600, 3)).astype(np.float32)
    # large-exponent coordinates (f32 box-distance overflow guard)
    cases["huge_coords_2d"] = (rng.standard_normal((300, 2)) * 1e30).astype(np.float32)
    cases["tiny_coords_3d"] = (rng.standard_normal((300, 3)) * 1e-30).astype(np.float32)
    cases["single_point"] = np.float32([[4.0, 5.0]])
    return cases


def _generated_inputs(emst):
    specs = {
        "uniform2d_1000_s0": ("uniform", 1000, 2, 0, {}),
        "normal3d_1000_s1": ("normal", 1000, 3, 1, {}),
        "blobs3d_3000_s2": ("blobs", 3000, 3, 2, {}),
        "blobs2d_3000_s3": ("blobs", 3000, 2, 3, {}),
        "uniform3d_5000_s4": ("uniform", 5000, 3, 4, {}),
        "normal2d_2000_s5": ("normal", 2000, 2, 5, {}),
        "blobs2d_tie_20000": ("blobs", 20000, 2, 0, {"blobs": 64, "spread": 0.002}),
        "blobs3d_1024_20000": ("blobs", 20000, 3, 1, {"blobs": 1024, "spread": 0.005}),
    }
    out = {}
    for name, (kind, n, d, seed, kw) in specs.items():
        out[name] = emst.generate(emst.DatasetSpec(kind, n, d, seed=seed, **kw))
    return out, specs


def _record_build(emst, pts, arrays, prefix):
    tree = emst.build(pts)
    codes = emst.morton_codes(pts)
    arrays[prefix + "codes"] = codes
    arrays[prefix + "perm"] = tree.leaf_perm
    arrays[prefix + "left"] = tree.left
    arrays[prefix + "right"] = tree.right
    arrays[prefix + "parent"] = tree.parent
    arrays[prefix + "leaf_parent"] = tree.leaf_parent
    arrays[prefix + "box_lo"] = tree.box_lo
    arrays[prefix + "box_hi"] = tree.box_hi
    return tree


def _record_rounds(emst, pts, tree, arrays, prefix, max_rounds=64):
    """Per-round intermediate state through the public building blocks (mst.py:436-547)."""
    state = emst.ComponentState.initial(tree)
    metric = emst.Euclidean()
    k = 0
    while len(np.unique(state.labels)) > 1 and k < max_rounds:
        p = f"{prefix}r{k}_"
        arrays[p + "labels_in"] = state.labels.copy()
        emst.reduce_labels(tree, state)
        arrays[p + "internal_labels"] = state.internal_labels.copy()
        emst.compute_upper_bounds(state, tree.leaf_perm, pts, metric)
        arrays[p + "upper_bounds"] = state.upper_bounds.copy()
        out = emst.find_component_outgoing_edges(tree, pts, state, metric)
        arrays[p + "reps"] = out.reps.copy()
        arrays[p + "best_u"] = out.u[out.reps].copy()
        arrays[p + "best_v"] = out.v[out.reps].copy()
        arrays[p + "best_w"] = out.w[out.reps].copy()
        res = emst.merge_components(state, out)
        arrays[p + "edge_u"] = res.edge_u
        arrays[p + "edge_v"] = res.edge_v
        arrays[p + "edge_w"] = res.edge_w
        arrays[p + "new_reps"] = res.new_reps
        arrays[p + "labels_out"] = state.labels.copy()
        k += 1
    return k


def make_small():
    emst = _import_reference()
    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"cases": {}, "matrix": {}, "generated": {}}

    ties = _tie_inputs()
    gen, specs = _generated_inputs(emst)
    for name, pts in list(ties.items()) + list(gen.items()):
        arrays[name + "/points"] = pts
        rec = {"n": int(pts.shape[0]), "d": int(pts.shape[1])}
        if name in specs:
            kind, n, d, seed, kw = specs[name]
            rec["spec"] = {"kind": kind, "n": n, "d": d, "seed": seed, **kw}
            rec["points_digest"] = array_digest(pts)
        tree = _record_build(emst, pts, arrays, name + "/")
        res = emst.boruvka_emst(pts)
        arrays[name + "/edges"] = res.edges
        arrays[name + "/weights"] = res.weights
        rec.update(_mst_record(res))
        # flags change work, never output (mst.py:601-607): record the no-opt eval count
        res_noopt = emst.boruvka_emst(pts, subtree_skip=False, upper_bound_seeding=False)
        assert np.array_equal(res_noopt.edges, res.edges)
        rec["leaf_distance_evals_noopt"] = int(res_noopt.leaf_distance_evals)
        if pts.shape[0] >= 2:
            rec["rounds"] = _record_rounds(emst, pts, tree, arrays, name + "/")
        meta["cases"][name] = rec

    # SPEC criterion-1 matrix (test_acceptance.py:54-78): digests only
    for kind in ("uniform", "normal", "blobs"):
        for d in (2, 3):
            for n in (1, 2, 10, 100, 1000, 2000):
                for seed in range(5):
                    pts = emst.generate(emst.DatasetSpec(kind, n, d, seed=seed))
                    res = emst.boruvka_emst(pts)
                    key = f"{kind}_{d}d_{n}_s{seed}"
                    rec = _mst_record(res)
                    rec["points_digest"] = array_digest(pts)
                    meta["matrix"][key] = rec

    # Morton KATs (test_geometry.py:108-119)
    unit2 = emst.Aabb(np.zeros(2), np.ones(2))
    unit3 = emst.Aabb(np.zeros(3), np.ones(3))
    meta["morton_kats"] = {
        "corner2_lo": emst.morton_encode((0.0, 0.0), unit2),
        "corner3_lo": emst.morton_encode((0.0, 0.0, 0.0), unit3),
        "corner2_hi": emst.morton_encode((1.0, 1.0), unit2),
        "corner3_hi": emst.morton_encode((1.0, 1.0, 1.0), unit3),
        "clamp2_lo": emst.morton_encode((-5.0, -5.0), unit2),
        "clamp2_hi": emst.morton_encode((5.0, 5.0), unit2),
    }

    np.savez_compressed(os.path.join(HERE, "small.npz"), **arrays)
    with open(os.path.join(HERE, "small.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote", len(arrays), "arrays and", len(meta["matrix"]), "matrix digests")


LARGE = {
    # BASELINE.json configs (SURVEY.md §8d inputs) plus the 1M survey goldens
    "uniform3d_100k": ("uniform", 100_000, 3, 0),
    "uniform3d_1m": ("uniform", 1_000_000, 3, 0),
    "blobs3d_1m": ("blobs", 1_000_000, 3, 0),
    "blobs2d_1m": ("blobs", 1_000_000, 2, 0),
    "normal3d_1m": ("normal", 1_000_000, 3, 0),
    "uniform2d_10m": ("uniform", 10_000_000, 2, 0),
    "normal3d_10m": ("normal", 10_000_000, 3, 0),
    "blobs2d_24m": ("blobs", 24_000_000, 2, 0),
    "blobs3d_37m": ("blobs", 37_000_000, 3, 0),
}


def make_large(names=None):
    emst = _import_reference()
    path = os.path.join(HERE, "large.json")
    meta = json.load(open(path)) if os.path.exists(path) else {}
    emst.boruvka_emst(emst.generate(emst.DatasetSpec("uniform", 300, 3, seed=0)))
    for name, (kind, n, d, seed) in LARGE.items():
        if names and name not in names:
            continue
        if name in meta:
            continue
        pts = emst.generate(emst.DatasetSpec(kind, n, d, seed=seed))
        tree = emst.build(pts)
        t0 = time.perf_counter()
        res = emst.boruvka_emst(pts)
        dt = time.perf_counter() - t0
        rec = _mst_record(res)
        rec.update({
            "spec": {"kind": kind, "n": n, "d": d, "seed": seed},
            "points_digest": array_digest(pts),
            "perm_digest": array_digest(tree.leaf_perm.astype("<i8")),
            "left_digest": array_digest(tree.left.astype("<i8")),
            "right_digest": array_digest(tree.right.astype("<i8")),
            "box_digest": array_digest(np.concatenate([tree.box_lo, tree.box_hi], 1)),
            "codes_digest": array_digest(emst.morton_codes(pts).astype("<u8")),
            "ref_seconds_survey_host": dt,
            "ref_phase_timings": res.phase_timings,
        })
        meta[name] = rec
        del tree, res, pts
        with open(path, "w") as fh:
            json.dump(meta, fh, indent=1, sort_keys=True)
        print(name, rec["iterations"], rec["total_weight"], rec["digest"], f"{dt:.1f}s", flush=True)


def make_mrd():
    """Mutual reachability: core distances and MSTs for k_pts in {2, 4, 16} (criteria 2 and 6)."""
    emst = _import_reference()
    arrays, meta = {}, {"cases": {}}
    cases = []
    for kind in ("uniform", "normal", "blobs"):
        for d in (2, 3):
            for n, seed in ((2, 0), (10, 1), (100, 2), (1000, 3), (5000, 4)):
                cases.append((kind, n, d, seed))
    cases.append(("blobs", 20000, 3, 5))
    cases.append(("blobs", 20000, 2, 6))
    for kind, n, d, seed in cases:
        pts = emst.generate(emst.DatasetSpec(kind, n, d, seed=seed))
        tree = emst.build(pts)
        name = f"{kind}{d}d_{n}_s{seed}"
        arrays[name + "/points"] = pts
        for k in (2, 4, 16):
            if k > n:
                continue
            core = emst.compute_core_distances(tree, pts, k).values
            res = emst.boruvka_emst(pts, metric="mrd", k_pts=k)
            key = f"{name}/k{k}"
            arrays[key + "/core"] = core
            arrays[key + "/edges"] = res.edges
            arrays[key + "/weights"] = res.weights
            rec = _mst_record(res)
            rec["core_digest"] = array_digest(core.astype("<f8"))
            meta["cases"][key] = rec
        print(name, flush=True)
    # a caller-given core table (MutualReachability(CoreDistances)) that is not a k-NN table
    pts = emst.generate(emst.DatasetSpec("normal", 3000, 3, seed=7))
    rng = np.random.default_rng(7)
    core = rng.random(3000) * 0.3
    arrays["given/points"] = pts
    arrays["given/core"] = core
    res = emst.boruvka_emst(pts, metric=emst.MutualReachability(emst.CoreDistances(4, core)))
    arrays["given/edges"] = res.edges
    arrays["given/weights"] = res.weights
    meta["cases"]["given"] = _mst_record(res)
    np.savez_compressed(os.path.join(HERE, "mrd.npz"), **arrays)
    with open(os.path.join(HERE, "mrd.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)


def _api_walks(emst, tree, pts, arrays, prefix):
    """traverse_nearest / for_each_leaf_to_root call sequences for a few queries (bvh.py:343-440)."""
    rng = np.random.default_rng(7)
    qs = np.concatenate([pts[rng.integers(0, pts.shape[0], 4)].astype(np.float64),
                         rng.random((2, pts.shape[1])) * 2 - 1])
    arrays[prefix + "queries"] = qs
    for j, q in enumerate(qs):
        seen = []

        def on_leaf(p, dist):
            seen.append((p, dist))
            return dist if dist > 0 else None   # nearest-neighbour shrink (ties stay visited)

        r = emst.traverse_nearest(tree, pts, q, on_leaf=on_leaf)
        arrays[prefix + f"walk{j}_pts"] = np.array([p for p, _ in seen], np.int64)
        arrays[prefix + f"walk{j}_dist"] = np.array([d for _, d in seen], np.float64)
        arrays[prefix + f"walk{j}_radius"] = np.array([r])
        pruned = []

        def prune(ref, lb, radius):
            pruned.append((ref, lb))
            return lb > 0.25 * (1 + (ref % 3))

        got = []
        r = emst.traverse_nearest(tree, pts, q, on_leaf=lambda p, d: got.append(p), prune=prune, radius=0.5)
        arrays[prefix + f"prune{j}_refs"] = np.array([a for a, _ in pruned], np.int64)
        arrays[prefix + f"prune{j}_lbs"] = np.array([b for _, b in pruned], np.float64)
        arrays[prefix + f"prune{j}_pts"] = np.array(got, np.int64)
    order = []
    emst.for_each_leaf_to_root(tree, lambda v: order.append(v))
    arrays[prefix + "sweep_visits"] = np.array(order, np.int64)
    stop = []
    emst.for_each_leaf_to_root(tree, lambda v: (stop.append(v), v % 5 != 0)[1])
    arrays[prefix + "sweep_visits_stop"] = np.array(stop, np.int64)


def make_api():
    """Goldens of the tree-level public API around the hot path: the level schedule
    (Bvh.sweep_order / sweep_starts), morton_codes / sort_by_morton with caller bounds, morton_encode,
    traverse_nearest and for_each_leaf_to_root call sequences."""
    emst = _import_reference()
    arrays = {}
    gen, _ = _generated_inputs(emst)
    cases = dict(_tie_inputs())
    cases.update({k: gen[k] for k in ("uniform2d_1000_s0", "normal3d_1000_s1", "blobs3d_3000_s2", "blobs2d_3000_s3")})
    names = []
    for name, pts in cases.items():
        if pts.shape[0] < 2:
            continue
        names.append(name)
        p = name + "/"
        tree = emst.build(pts)
        arrays[p + "points"] = pts
        for f in ("leaf_perm", "left", "right", "parent", "leaf_parent", "box_lo", "box_hi"):
            arrays[p + f] = getattr(tree, f)
        arrays[p + "sweep_order"] = tree.sweep_order
        arrays[p + "sweep_starts"] = tree.sweep_starts
        d = pts.shape[1]
        lo, hi = pts.min(0).astype(np.float64), pts.max(0).astype(np.float64)
        ext = hi - lo
        for tag, blo, bhi in (("inner", lo + 0.25 * ext, hi - 0.3 * ext), ("outer", lo - 1.5, hi + 0.75),
                              ("flat", np.where(np.arange(d) == 0, lo, lo - 1), np.where(np.arange(d) == 0, lo, hi + 1))):
            b = emst.Aabb(blo, bhi)
            arrays[p + f"bounds_{tag}"] = np.stack([blo, bhi])
            arrays[p + f"codes_{tag}"] = emst.morton_codes(pts, b)
            arrays[p + f"perm_{tag}"] = emst.sort_by_morton(pts, b)
            arrays[p + f"encode_{tag}"] = np.array([emst.morton_encode(x, b) for x in pts[:16]], np.uint64)
        if name in ("uniform2d_1000_s0", "normal3d_1000_s1", "grid9", "lattice_dups_3d"):
            _api_walks(emst, tree, pts, arrays, p)
    np.savez_compressed(os.path.join(HERE, "api.npz"), **arrays)
    with open(os.path.join(HERE, "api.json"), "w") as fh:
        json.dump({"cases": names}, fh, indent=1)


IO_EDGE_CASES = [
    "0,1,0.5\n1,2,0.25\n", "0,1,0.5\r\n1,2,0.25\r\n", "0,1,0.5\r1,2,0.25\r", "0,1,0.5", "", "\n \n\t\n",
    "\n\n0,1,2\n  \n\x0c\n3,4,5\n\x1c\n", "  1 , 2 ,  0.5  \n", "+1,2,3\n", "1_0,2,3.5\n", "1,2,1e-400\n",
    "1,2,1e400\n", "1,2,inf\n", "1,2,nan\n", "-1,2,3\n", "-0,2,3\n", "1,-2,3\n", "1,2\n", "1,2,3,4\n",
    "a,2,3\n", "1,2,3.5e\n", "\u00a01,2,3\n", "\uff11,2,3\n", "1,2,.5\n1,2,5.\n1,2,-0.0\n1,2,1E+3\n",
    "1,2,0x10\n", "1.0,2,3\n", "1,2,3\n\n5,6,bad\n7,8,9\n", "1,2,3\n4,5\n6,7,inf\n",
    "007,08,1.25e-3\n", "1,2,3 4\n", "1,,3\n", ",1,2\n", "1,2,\n", "1,2,3\r\n\r\n4,5,6", "1 2,3,4\n",
    "1,2,1e308\n3,4,2.2250738585072014e-308\n5,6,4.9e-324\n", "1,2,0.1000000000000000055511151231257827\n",
]
IO_POINT_CASES = [
    "0.5,0.25\n1,2\n", "0.5,0.25,1\n1,2,3\n", "1\n", "1,2,3,4\n", "1,2\n3,4,5\n", "1,2,3\n4,5\n",
    "1e39,2\n", "nan,1\n", "1,inf\n", "", "\n\n", "\n  \n1,2\n", "1_0,2\n", "a,b\n", "\u00a01,2\n",
    "1,2\r\n3,4\r\n", "1,2\r3,4", ".5,5.\n-0,+1e-3\n", "1,2,\n", "1, 2 ,3\n", "3.4028235677973366e38,1\n",
    "1e-50,1\n", "0.1,0.2,0.3\n0.4,0.5,bad\n",
]


def make_io():
    """The reference's CSV readers on edge cases (line endings, whitespace, Python-only spellings, every
    error): each input is written as UTF-8 to a file and read back through the reference's read_edges /
    read_points (data.py:148-198, 225-257); the outputs or the exception (type and message) are recorded."""
    import tempfile
    emst = _import_reference()
    out = {"edges": [], "points": []}
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "case.csv")
        for kind, cases in (("edges", IO_EDGE_CASES), ("points", IO_POINT_CASES)):
            for text in cases:
                with open(path, "wb") as fh:
                    fh.write(text.encode("utf-8"))
                rec = {"text": text}
                try:
                    if kind == "edges":
                        e, w = emst.read_edges(path)
                        rec["edges"] = e.tolist()
                        rec["weights_hex"] = [float(x).hex() for x in w]
                    else:
                        p = emst.read_points(path)
                        rec["shape"] = list(p.shape)
                        rec["points_hex"] = [float(x).hex() for x in p.reshape(-1)]
                except Exception as exc:   # the reference's exception is part of the contract
                    rec["error"] = type(exc).__name__
                    rec["message"] = str(exc)
                out[kind].append(rec)
    with open(os.path.join(HERE, "io_cases.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "small"
    if which == "small":
        make_small()
    elif which == "io":
        make_io()
    elif which == "api":
        make_api()
    elif which == "mrd":
        make_mrd()
    else:
        make_large(sys.argv[2:] or None)
