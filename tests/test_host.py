"""CPU-side checks of the drop-in boundary: the C ABI library, validation, errors, no CPU fallback."""

import ctypes
import os
import re

import numpy as np
import pytest
import torch

import paper_2207_00514_b200 as E
from paper_2207_00514_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "emst_b200.h")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(emst_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    names = _declared()
    assert "emst_boruvka" in names and len(names) >= 12
    for name in names:
        assert hasattr(L, name), name
    assert set(_lib.EXPORTS) == set(names)


def test_library_is_built_for_sm100a():
    assert b"sm_100a" in _lib.load().emst_build_info()
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_stats_struct_matches_header(tmp_path):
    """emst_stats: every ctypes field sits at the C compiler's offset for include/emst_b200.h."""
    import subprocess
    names = [f[0] for f in _lib.Stats._fields_]
    src = tmp_path / "layout.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "emst_b200.h"\nint main(void) {\n'
                   + "".join(f'  printf("%zu\\n", offsetof(emst_stats, {n}));\n' for n in names)
                   + '  printf("%zu\\n", sizeof(emst_stats));\n  return 0;\n}\n')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    want = [getattr(_lib.Stats, n).offset for n in names] + [ctypes.sizeof(_lib.Stats)]
    assert got == want


def test_exception_names_match_reference():
    names = ["EmstError", "EmptyDatasetError", "InvalidCoordinateError", "DimensionMismatchError",
             "UnsupportedDimensionError", "InvalidParameterError", "InvalidIndexError", "ParseError",
             "OracleCapError", "NoOutgoingEdgeError", "NothingToFindError", "TraversalStackOverflowError",
             "InternalInvariantViolation"]
    for n in names:
        cls = getattr(E, n)
        assert issubclass(cls, E.EmstError)
    assert issubclass(E.DeviceError, E.EmstError)


def test_parameter_validation_precedes_device_work():
    """mst.py:609-617 order: k_pts type / range, metric, euclidean k_pts, threads -- no GPU touched."""
    pts = np.zeros((10, 2), np.float32)
    with pytest.raises(E.InvalidParameterError):
        E.boruvka_emst(pts, metric="chebyshev")
    with pytest.raises(E.InvalidParameterError):
        E.boruvka_emst(pts, metric="euclidean", k_pts=3)
    with pytest.raises(E.InvalidParameterError):
        E.boruvka_emst(pts, metric="mrd", k_pts=0)
    with pytest.raises(E.InvalidParameterError):
        E.boruvka_emst(pts, k_pts=True)
    with pytest.raises(E.InvalidParameterError):
        E.boruvka_emst(pts, threads=-1)
    with pytest.raises(E.InvalidParameterError):
        E.boruvka_emst(pts, threads=1.5)


def test_shape_validation_on_host():
    with pytest.raises(E.EmptyDatasetError):
        E.as_point_array(np.empty((0, 2)))
    with pytest.raises(E.UnsupportedDimensionError):
        E.as_point_array(np.zeros((4, 5)))
    with pytest.raises(E.UnsupportedDimensionError):
        E.as_point_array(np.zeros(4))
    with pytest.raises(E.InvalidCoordinateError, match="point 1 "):
        E.as_point_array([[0.0, 0.0], [np.inf, 0.0]])
    out = E.as_point_array([[0, 1], [2, 3]])
    assert out.dtype == np.float32 and out.flags.c_contiguous


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu():
    with pytest.raises(E.DeviceError):
        E.boruvka_emst(np.random.default_rng(0).random((100, 3)).astype(np.float32))


def test_weighted_edge_order():
    e = E.WeightedEdge(5, 2, 1.5)
    assert (e.u, e.v) == (2, 5)
    assert E.WeightedEdge(1, 2, 1.0) < E.WeightedEdge(1, 3, 1.0) < E.WeightedEdge(0, 1, 2.0)
    with pytest.raises(E.InvalidParameterError):
        E.WeightedEdge(3, 3, 0.0)


def test_geometry_helpers():
    assert E.distance([0, 0], [3, 4]) == 5.0
    box = E.Aabb(np.zeros(2), np.ones(2))
    assert E.distance_point_box([2.0, 0.5], box) == 1.0
    assert E.distance_point_box([0.5, 0.5], box) == 0.0


def test_oracle_is_not_imported_by_the_product():
    import pathlib
    for path in pathlib.Path(ROOT, "paper_2207_00514_b200").rglob("*.py"):
        assert "oracle" not in path.read_text().replace("Oracle", ""), path


def test_run_bench_validates_before_any_gpu_work():
    pts = E.generate(E.DatasetSpec("uniform", 100, 2, seed=0))
    with pytest.raises(E.EmstError):
        E.run_bench(pts, [10], repeats=0)
