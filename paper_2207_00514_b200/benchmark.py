"""``run_bench``: the paper's scaling methodology on the GPU.

The reference's ``emst bench`` (cli.py:63-104) times the
engine on seeded subsamples of growing size and reports one tab-separated row
per size: medians over ``repeats`` runs of the phase timings, the rate
n * d / t_total and the growth of t_total from the previous size.  The rows,
columns and errors are the reference's; the runs are ``boruvka_emst`` on the
B200.  ``resident=True`` hands each subsample over as a CUDA tensor once, so
the rows time the device-resident solve (the bench.py ``value`` path) instead
of the host-pointer entry with its PCIe copies.
"""

from __future__ import annotations

import statistics
from dataclasses import dataclass

import numpy as np

from .data import sample
from .errors import EmstError
from .mst import boruvka_emst

# (column header, BenchReport field, formatter): the row layout of cli.py:44-61
_G9 = "{:.9g}".format
_COLUMNS = (
    ("dataset", "dataset", str), ("n", "n", str), ("d", "d", str), ("metric", "metric", str),
    ("k_pts", "k_pts", str), ("threads", "threads", str), ("repeats", "repeats", str),
    ("iterations", "iterations", str), ("leaf_evals", "leaf_distance_evals", str),
    ("t_tree", "t_tree", _G9), ("t_core", "t_core", _G9), ("t_mst", "t_mst", _G9),
    ("t_total", "t_total", _G9), ("rate", "rate", _G9), ("time_ratio_prev", "time_ratio_prev", _G9),
)


@dataclass
class BenchReport:
    """One size's row: medians over the repeats (fields of cli.py:28-43)."""

    dataset: str
    n: int
    d: int
    metric: str
    k_pts: int
    threads: int
    repeats: int
    iterations: int
    leaf_distance_evals: int
    t_tree: float
    t_core: float
    t_mst: float
    t_total: float
    rate: float
    time_ratio_prev: float

    HEADER = "\t".join(head for head, _, _ in _COLUMNS)

    def row(self) -> str:
        return "\t".join(fmt(getattr(self, name)) for _, name, fmt in _COLUMNS)


_PHASES = ("tree", "core", "mst", "total")


def _one_size(dataset, pts, m, d, repeats, solve, metric, k_pts) -> tuple[BenchReport, float]:
    runs = [solve(pts) for _ in range(repeats)]
    med = {p: statistics.median(r.phase_timings[p] for r in runs) for p in _PHASES}
    first = runs[0]
    rep = BenchReport(dataset, m, d, metric, k_pts, first.threads, repeats, first.iterations,
                      first.leaf_distance_evals, med["tree"], med["core"], med["mst"], med["total"],
                      m * d / med["total"] if med["total"] > 0 else float("inf"), float("nan"))
    return rep, med["total"]


def run_bench(points, sizes, *, repeats: int = 3, metric: str = "euclidean", k_pts: int = 1, threads: int = 0,
              dataset: str = "points", seed: int = 0, resident: bool = False) -> list[BenchReport]:
    """One BenchReport per entry of `sizes` (cli.py:63-104 semantics).

    Size i uses the seeded subsample ``sample(points, m, seed + 1 + i)`` (the whole
    cloud when m == n); a 256-point run first absorbs the one-time setup (context
    creation, workspace allocation) the way the reference's warm-up absorbs JIT
    loading.  Errors: repeats < 1 and sizes outside [1, n] raise EmstError.
    """
    if repeats < 1:
        raise EmstError(f"repeats must be >= 1, got {repeats}")
    cloud = np.asarray(points)
    n, d = cloud.shape
    for m in sizes:   # (validated up front: no GPU work for a bad request)
        if not 1 <= m <= n:
            raise EmstError(f"sample size {m} out of range for {n} points")

    def solve(pts):
        return boruvka_emst(pts, metric=metric, k_pts=k_pts, threads=threads)

    warm = sample(cloud, min(n, 256), seed)
    boruvka_emst(warm, metric=metric, k_pts=min(k_pts, warm.shape[0]), threads=threads)
    reports: list[BenchReport] = []
    for i, m in enumerate(sizes):
        pts = cloud if m == n else sample(cloud, m, seed + 1 + i)
        if resident:
            import torch
            pts = torch.from_numpy(np.ascontiguousarray(pts, dtype=np.float32)).cuda()
        rep, total = _one_size(dataset, pts, m, d, repeats, solve, metric, k_pts)
        if reports and reports[-1].t_total:
            rep.time_ratio_prev = total / reports[-1].t_total
        reports.append(rep)
    return reports

