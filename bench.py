#!/usr/bin/env python
"""EMST throughput on B200: MFeatures/s = n*d / t / 1e6 (reference cli.py:100).

One "step" is one full ``boruvka_emst`` of the synthetic cloud (build + all
Boruvka rounds + final (w, u, v) edge sort), points resident in HBM before the
timed region (``value``) or handed over as a plain numpy array with the edges
read back inside it (``e2e``, through the public drop-in API).  The output of
the timed run is digested and compared with the reference's (``parity``).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config blobs3d_37m] [--impl ours|reference]

N > 1 runs one process per GPU (under torchrun; without it bench.py relaunches
itself through torchrun): every rank builds the same tree and takes a Morton
slot range of each round's traversal; per-component minima meet in a
two-phase NCCL min-allreduce (strong scaling: total work fixed).
``--impl reference`` times the reference algorithm's CPU implementation (the C
restatement in oracle/, all host threads) on the same whole cloud.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

# BASELINE.json configs: name -> (kind, n, d, seed)
CONFIGS = {
    "blobs3d_37m": ("blobs", 37_000_000, 3, 0),     # configs[3], the headline (HACC-like)
    "blobs2d_24m": ("blobs", 24_000_000, 2, 0),     # configs[4] (GeoLife-like)
    "uniform2d_10m": ("uniform", 10_000_000, 2, 0), # configs[1]
    "normal3d_10m": ("normal", 10_000_000, 3, 0),   # configs[2]
    "uniform3d_100k": ("uniform", 100_000, 3, 0),   # configs[0]
}
METRIC = "MFeatures/s for EMST of 37M-pt 3D synthetic cloud, 1/2/4/8 B200; HBM GB/s"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0   # GB/s, /opt/skills/guides/B200_PROFILING.md fallback

_THROTTLE = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
             0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}


def hbm_peak():
    try:
        with open(PEAKS_PATH) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


TRAFFIC_PATH = os.path.join(ROOT, "profiles", "r02_traverse_traffic.json")


def measured_traffic(cfg: str):
    """DRAM bytes per traversal launch from the committed ncu capture of this config (profiles/), or None."""
    try:
        with open(TRAFFIC_PATH) as fh:
            return float(json.load(fh)[cfg]["dram_bytes_per_launch"])
    except Exception:
        return None


def algorithmic_bytes(n: int, d: int, counts: list[int]) -> float:
    """(24d+72)n + K(16d+84)n + 56*sum(c_k) + 48(n-1)."""
    rounds = len(counts) - 1
    return (24 * d + 72) * n + rounds * (16 * d + 84) * n + 56 * sum(counts[:-1]) + 48 * (n - 1)


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling (NVML) during the timed region."""

    def __init__(self, device: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in _THROTTLE.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.1)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def make_points(cfg: str):
    import paper_2207_00514_b200 as E
    kind, n, d, seed = CONFIGS[cfg]
    return E.generate(E.DatasetSpec(kind, n, d, seed))


def cpu_sample(points, m: int):
    import paper_2207_00514_b200 as E
    return E.sample(points, min(m, points.shape[0]), 0)


def run_reference(args):
    """The reference arm: the reference algorithm's CPU implementation on the headline cloud itself.

    Every timed step is one full solve of the whole config (same n, d, seed as our arm, so the
    driver's ratio compares like with like).  The C restatement runs on all host threads; it needs
    no JIT, so the W warm-up steps touch the code and memory on a 1M-point sample instead of
    repeating full 37M solves.  Timed steps stop early (reported as `steps_timed`) if they would run
    past --ref-budget seconds.
    """
    world, rank, _ = dist_env()
    cfg = args.config
    kind, n, d, seed = CONFIGS[cfg]
    if rank != 0:
        return
    from oracle import oracle as orc
    pts = make_points(cfg)
    orc.set_threads(os.cpu_count() or 1)
    threads = orc.num_threads()
    warm = cpu_sample(pts, min(1_000_000, n))
    for _ in range(args.warmup):
        orc.boruvka_emst(warm)
    times = []
    t_begin = time.perf_counter()
    for i in range(args.steps):
        t0 = time.perf_counter()
        res = orc.boruvka_emst(pts)
        times.append(time.perf_counter() - t0)
        spent = time.perf_counter() - t_begin
        if spent + statistics.median(times) > args.ref_budget and i + 1 < args.steps:
            break
    dt = statistics.median(times)
    value = n * d / dt / 1e6
    sample = f"the whole {cfg} cloud (n={n}) per step, {threads} OpenMP threads"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "MFeatures/s", "n_gpus": args.gpus,
        "steps": args.steps, "steps_timed": len(times), "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32 coords / f64 weights",
        "data": "synthetic (reference generator, seed 0)",
        "config": {"workload": cfg, "kind": kind, "n": n, "d": d, "seed": seed,
                   "warmup_sample_points": warm.shape[0]},
        "cpu_baseline": {"value": value, "unit": "MFeatures/s", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "MFeatures/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "parity": parity_record(cfg, res.edges, res.weights),
    }
    print(json.dumps(line), flush=True)


def parity_record(cfg: str, edges, weights) -> dict:
    """sha256(edges || weights)[:16] of a run's output against the reference's own (tests/golden/large.json)."""
    import hashlib
    e = np.ascontiguousarray(edges, dtype="<i8")
    w = np.ascontiguousarray(weights, dtype="<f8")
    got = hashlib.sha256(e.tobytes() + w.tobytes()).hexdigest()[:16]
    want = None
    try:
        with open(os.path.join(ROOT, "tests", "golden", "large.json")) as fh:
            want = json.load(fh)[cfg]["digest"]
    except Exception:
        pass
    return {"digest": got, "reference_digest": want, "ok": want is not None and got == want}


def setup_ranks(world: int, rank: int, local: int):
    """(context, torch.distributed module or None, description) for this rank.

    One process per GPU over NCCL when there are enough GPUs; with fewer GPUs than
    ranks (a single-GPU box) the ranks share devices and exchange through the host
    (gloo) -- the same sharded traversal and exchange kernels, another transport.
    """
    import torch
    import paper_2207_00514_b200 as E
    from paper_2207_00514_b200 import distributed as D

    if world == 1:
        torch.cuda.set_device(local)
        return E.Context(local), None, {"devices": 1, "exchange": "none"}
    import torch.distributed as dist
    ndev = torch.cuda.device_count()
    if ndev >= world:
        device = local
        torch.cuda.set_device(device)
        dist.init_process_group("nccl", device_id=torch.device("cuda", device))
        exchange = "nccl"
    else:
        device = local % ndev
        torch.cuda.set_device(device)
        dist.init_process_group("gloo")
        exchange = "host"
    ctx = D.init_context(device=device, exchange=exchange)
    desc = {"devices": min(ndev, world), "exchange": exchange}
    if exchange == "host":
        desc["note"] = f"{world} ranks share {ndev} GPU(s): host (gloo) exchange; not a scaling measurement"
    return ctx, dist, desc


def max_over_ranks(dist, x: float) -> float:
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_ours(args):
    import torch
    import paper_2207_00514_b200 as E

    world, rank, local = dist_env()
    cfg = args.config
    kind, n, d, seed = CONFIGS[cfg]
    ctx, dist, ranks = setup_ranks(world, rank, local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream)

    pts_host = make_points(cfg)
    pts_dev = torch.from_numpy(pts_host).cuda()
    edges = torch.empty((n - 1, 2), dtype=torch.int64, device="cuda")
    weights = torch.empty((n - 1,), dtype=torch.float64, device="cuda")

    def step():
        return E.boruvka_emst_device(pts_dev, edges, weights, context=ctx)

    if args.profile:
        step()
        torch.cuda.synchronize()
        return

    for _ in range(args.warmup):
        st = step()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    trav_ms = trav_launch = launches = 0
    with ClockSampler(torch.cuda.current_device()) as clocks:
        start.record(stream)
        for _ in range(args.steps):
            st = step()
            trav_ms += st.traverse_ms
            trav_launch += st.traverse_launches
            launches += st.kernel_launches
        end.record(stream)
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ms = max_over_ranks(dist, start.elapsed_time(end) / args.steps)
    value = n * d / (ms / 1e3) / 1e6
    counts = [int(st.component_counts[i]) for i in range(st.num_counts)]
    # parity of the exact run just timed: the last step's device-resident output against the reference
    parity = parity_record(cfg, edges.cpu().numpy(), weights.cpu().numpy())
    del pts_dev

    # end to end through the public drop-in as a caller uses it: a plain (pageable) numpy array in,
    # numpy edges / weights out, every copy inside the timed region
    e2e_ms = []
    for i in range(max(2, min(args.steps, 3)) + 1):
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = E.boruvka_emst(pts_host, context=ctx)
        dt = (time.perf_counter() - t0) * 1e3
        if i > 0:
            e2e_ms.append(dt)
    e2e = max_over_ranks(dist, statistics.median(e2e_ms))
    assert res.component_counts == counts
    e2e_parity = parity_record(cfg, res.edges, res.weights)

    peak, peak_src = hbm_peak()
    # dominant kernel: the traversal; algorithmic bytes per query per round = 12d + 36
    per_step_trav_ms = trav_ms / args.steps
    trav_bytes = (12 * d + 36) * st.traverse_queries
    trav_gbs = trav_bytes / (st.traverse_ms / 1e3) / 1e9 if st.traverse_ms > 0 else 0.0
    whole_bytes = algorithmic_bytes(n, d, counts)
    # every rank's phase times (the replicated phases bound the multi-GPU speed-up)
    phases = {k: round(st.phase_ms[i], 3) for i, k in enumerate(E._lib.PHASES)}
    rank_phases = [phases]
    if dist is not None:
        rank_phases = [None] * world
        dist.all_gather_object(rank_phases, phases)
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": value, "unit": "MFeatures/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32 coords / f64 weights", "data": "synthetic (reference generator, seed 0)",
        "config": {"workload": cfg, "kind": kind, "n": n, "d": d, "seed": seed,
                   "parallelism": f"replicated tree, traversal sharded by Morton range x{world}", **ranks,
                   "l2": "inputs larger than L2 (points 444 MB + 2.4 GB tree at 37M), no flush"},
        "parity": parity,
        "e2e": {"value": n * d / (e2e / 1e3) / 1e6, "unit": "MFeatures/s", "ms_per_step": e2e,
                "input": "pageable numpy array through boruvka_emst", "parity_ok": e2e_parity["ok"],
                "h2d_bytes_per_step": n * d * 4, "d2h_bytes_per_step": (n - 1) * 24},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "kernel": "k_traverse", "achieved": trav_gbs, "peak": peak, "unit": "GB/s",
                     "frac": trav_gbs / peak, "traffic": measured_traffic(cfg),
                     "traffic_source": "ncu dram__bytes_read.sum + dram__bytes_write.sum per k_traverse launch "
                                       f"({os.path.relpath(TRAFFIC_PATH, ROOT)})",
                     "algorithmic_bytes_per_launch": trav_bytes / max(st.traverse_launches, 1),
                     "peak_source": peak_src,
                     "bytes_model": f"(12d+36) B per query per round = {12 * d + 36} B",
                     "launches_per_step": st.traverse_launches, "ms_per_step": per_step_trav_ms},
        "whole_step_roofline": {"algorithmic_bytes": whole_bytes, "achieved_gbs": whole_bytes / (ms / 1e3) / 1e9,
                                "frac": whole_bytes / (ms / 1e3) / 1e9 / (peak * world)},
        "iterations": int(st.iterations), "component_counts": counts,
        "rounds": [{"traverse_ms": round(st.round_traverse_ms[i], 3), "node_visits": int(st.round_node_visits[i]),
                    "found": int(st.round_found[i]), "skipped": int(st.round_skipped[i])} for i in range(min(st.iterations, 64))],
        "phase_ms": phases,
        "rank_phase_ms": rank_phases if world > 1 else None,
        "clocks": clocks.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as orc
        orc.set_threads(os.cpu_count() or 1)
        t0 = time.perf_counter()
        orc.boruvka_emst(pts_host)
        dt = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": n * d / dt / 1e6, "unit": "MFeatures/s", "cores": orc.num_threads(),
                                "kind": "port", "sample": f"the whole {cfg} cloud (n={n}), one solve, {dt:.1f} s"}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` outside torchrun: relaunch this script as N ranks (torchrun, 127.0.0.1)."""
    import socket
    import subprocess
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")   # (stderr: lets the driver see the N ranks come up)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="blobs3d_37m", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-budget", type=float, default=1200.0,
                    help="reference arm: stop timing full solves after about this many seconds")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true", help="one untimed step only (for ncu); prints nothing")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(spawn_ranks(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
