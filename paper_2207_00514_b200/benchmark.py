"""``run_bench`` on the GPU (reference cli.py:26-104).

The paper's scaling methodology: the engine at several
seeded subsample sizes, medians of ``repeats`` runs, rate = n * d / t_total
features per second.  Same arguments, report rows and errors as the reference;
the timings are the GPU path's phase timings (tree / core / mst / total).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .data import sample
from .errors import EmstError
from .mst import boruvka_emst


def _fmt(x: float) -> str:
    return f"{x:.9g}"


@dataclass
class BenchReport:
    """One benchmark row: medians of `repeats` runs at one size (cli.py:26-61)."""

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

    HEADER = "\t".join([
        "dataset", "n", "d", "metric", "k_pts", "threads", "repeats",
        "iterations", "leaf_evals", "t_tree", "t_core", "t_mst",
        "t_total", "rate", "time_ratio_prev",
    ])

    def row(self) -> str:
        return "\t".join([
            self.dataset, str(self.n), str(self.d), self.metric,
            str(self.k_pts), str(self.threads), str(self.repeats),
            str(self.iterations), str(self.leaf_distance_evals),
            _fmt(self.t_tree), _fmt(self.t_core), _fmt(self.t_mst),
            _fmt(self.t_total), _fmt(self.rate), _fmt(self.time_ratio_prev),
        ])


def run_bench(points, sizes, *, repeats: int = 3, metric: str = "euclidean", k_pts: int = 1, threads: int = 0,
              dataset: str = "points", seed: int = 0) -> list[BenchReport]:
    """Benchmark the engine at several subsample sizes (cli.py:63-104).

    Each size gets its own seeded subsample; medians are taken over `repeats`
    runs.  One small untimed run first absorbs one-time setup (context, workspace).
    """
    if repeats < 1:
        raise EmstError(f"repeats must be >= 1, got {repeats}")
    pts = np.asarray(points)
    n, d = pts.shape
    warm = sample(pts, min(n, 256), seed)
    boruvka_emst(warm, metric=metric, k_pts=min(k_pts, warm.shape[0]), threads=threads)
    reports: list[BenchReport] = []
    prev_total = None
    for idx, m in enumerate(sizes):
        if not 1 <= m <= n:
            raise EmstError(f"sample size {m} out of range for {n} points")
        sub = sample(pts, m, seed + 1 + idx) if m < n else pts
        runs = [boruvka_emst(sub, metric=metric, k_pts=k_pts, threads=threads) for _ in range(repeats)]
        t_tree = float(np.median([r.phase_timings["tree"] for r in runs]))
        t_core = float(np.median([r.phase_timings["core"] for r in runs]))
        t_mst = float(np.median([r.phase_timings["mst"] for r in runs]))
        t_total = float(np.median([r.phase_timings["total"] for r in runs]))
        reports.append(BenchReport(
            dataset=dataset, n=m, d=d, metric=metric, k_pts=k_pts, threads=runs[0].threads, repeats=repeats,
            iterations=runs[0].iterations, leaf_distance_evals=runs[0].leaf_distance_evals,
            t_tree=t_tree, t_core=t_core, t_mst=t_mst, t_total=t_total,
            rate=m * d / t_total if t_total > 0 else float("inf"),
            time_ratio_prev=t_total / prev_total if prev_total else float("nan"),
        ))
        prev_total = t_total
    return reports
