"""Point / edge files: formats byte-identical to the reference's writers.

The expected text is built with the reference's own per-row expressions
(data.py:126 ``",".join(f"{float(x):.9g}" for x in row)`` and data.py:211
``f"{int(u)},{int(v)},{float(w):.17g}\\n"``); the native formatter (csrc/textio.h)
must reproduce it exactly.  Host-only: no GPU needed.
"""

import io

import numpy as np
import pytest

import paper_2207_00514_b200 as E


def _ref_edges_text(edges, weights):
    return "".join(f"{int(u)},{int(v)},{float(w):.17g}\n" for (u, v), w in zip(edges, weights))


def _ref_points_text(pts):
    return "".join(",".join(f"{float(x):.9g}" for x in row) + "\n" for row in pts)


def test_write_edges_matches_reference_format():
    rng = np.random.default_rng(0)
    m = 50_000
    edges = np.stack([rng.integers(0, 2**31, m), rng.integers(0, 2**40, m)], 1).astype(np.int64)
    w = np.concatenate([rng.random(m // 4), rng.random(m // 4) * 1e-8, np.exp(rng.normal(size=m // 4) * 30),
                        rng.integers(0, 1000, m - 3 * (m // 4)).astype(np.float64)])
    w[:9] = [0.0, -0.0, 5e-324, 1.7976931348623157e308, 0.1, 1e16, 1e-5, 123456789012345678.0, 2.5e-5]
    buf = io.StringIO()
    E.write_edges(buf, edges, w)
    assert buf.getvalue() == _ref_edges_text(edges, w)


def test_write_points_matches_reference_format():
    for d in (2, 3):
        pts = E.generate(E.DatasetSpec("normal", 20_000, d, seed=d))
        pts[0, :2] = [1e-30, -3.4028235e38]
        buf = io.StringIO()
        E.write_points(buf, pts)
        assert buf.getvalue() == _ref_points_text(pts)


def test_edge_round_trip_is_lossless(tmp_path):
    pts = E.generate(E.DatasetSpec("blobs", 3000, 3, seed=0))
    from oracle import oracle as orc
    res = orc.boruvka_emst(pts)
    path = tmp_path / "edges.csv"
    E.write_edges(str(path), res.edges, res.weights)
    e, w = E.read_edges(str(path))
    assert np.array_equal(e, res.edges) and np.array_equal(w, res.weights)


def test_point_formats_round_trip(tmp_path):
    pts = E.generate(E.DatasetSpec("uniform", 1000, 2, seed=3))
    for fmt, prec in (("csv", 4), ("bin", 4), ("bin", 8)):
        path = tmp_path / f"p.{fmt}{prec}"
        E.write_points(str(path), pts, fmt=fmt, precision=prec)
        back = E.read_points(str(path), fmt=fmt)
        assert back.dtype == np.float32 and np.array_equal(back, pts), (fmt, prec)


def test_io_errors(tmp_path):
    with pytest.raises(E.InvalidParameterError):
        E.write_edges(io.StringIO(), np.zeros((3, 2), np.int64), np.zeros(2))
    with pytest.raises(E.InvalidParameterError):
        E.write_points(io.StringIO(), np.zeros((3, 2), np.float32), fmt="bin", precision=2)
    with pytest.raises(E.ParseError):
        E.read_edges(io.StringIO("1,2\n"))
    with pytest.raises(E.ParseError):
        E.read_edges(io.StringIO("1,2,inf\n"))
    with pytest.raises(E.ParseError):
        E.read_points(io.StringIO("1,2\n3,4,5\n"))
    with pytest.raises(E.EmptyDatasetError):
        E.read_points(io.StringIO("\n\n"))
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"XXXX" + bytes(20))
    with pytest.raises(E.ParseError):
        E.read_points(str(bad), fmt="bin")


def _io_cases():
    import json
    import os
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io_cases.json")) as fh:
        return json.load(fh)


@pytest.mark.parametrize("source", ["path", "textio"])
def test_readers_match_reference_on_edge_cases(tmp_path, source):
    """read_edges / read_points (native parser + the reference's per-line rules for the lines it hands back)
    against the reference's own readers on line-ending, whitespace, Python-only spellings and every error
    (tests/golden/make_goldens.py io)."""
    cases = _io_cases()
    for kind, reader in (("edges", E.read_edges), ("points", E.read_points)):
        for i, rec in enumerate(cases[kind]):
            path = tmp_path / f"{kind}{i}.csv"
            path.write_bytes(rec["text"].encode("utf-8"))
            src = str(path) if source == "path" else io.StringIO(rec["text"], newline=None)
            if source == "textio":   # a text stream already applies universal newlines, like the reference's open()
                src = io.StringIO(path.read_text())
            if "error" in rec:
                with pytest.raises(Exception) as info:
                    reader(src)
                assert type(info.value).__name__ == rec["error"], (kind, rec["text"])
                assert str(info.value) == rec["message"], (kind, rec["text"])
                continue
            if kind == "edges":
                e, w = reader(src)
                assert e.dtype == np.int64 and e.shape == (len(rec["edges"]), 2), rec["text"]
                assert e.tolist() == rec["edges"], rec["text"]
                assert [float(x).hex() for x in w] == rec["weights_hex"], rec["text"]
            else:
                p = reader(src)
                assert p.dtype == np.float32 and list(p.shape) == rec["shape"], rec["text"]
                assert [float(x).hex() for x in p.reshape(-1)] == rec["points_hex"], rec["text"]


def test_large_edge_file_reads_fast(tmp_path):
    """37M-edge files are the use case; 2M edges here must take well under a second
    of parsing, bit-exact through the %.17g round trip, with an error on the last line reported by number."""
    import time
    rng = np.random.default_rng(1)
    m = 2_000_000
    edges = np.stack([rng.integers(0, 2**31, m), rng.integers(0, 2**31, m)], 1).astype(np.int64)
    w = rng.random(m) * np.exp(rng.normal(size=m) * 5)
    path = tmp_path / "big.csv"
    E.write_edges(str(path), edges, w)
    t0 = time.perf_counter()
    e2, w2 = E.read_edges(str(path))
    dt = time.perf_counter() - t0
    assert np.array_equal(e2, edges) and np.array_equal(w2, w)
    assert dt < 5.0, dt
    with open(path, "a") as fh:
        fh.write("1,2,oops\n")
    with pytest.raises(E.ParseError, match=f"line {m + 1}: could not parse '1,2,oops'"):
        E.read_edges(str(path))
    pts = E.generate(E.DatasetSpec("normal", 1_000_000, 3, seed=2))
    E.write_points(str(tmp_path / "p.csv"), pts)
    assert np.array_equal(E.read_points(str(tmp_path / "p.csv")), pts)
