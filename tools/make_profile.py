"""Compose profiles/<round>_profile.md and refresh profiles/ from an evidence run in gpurun_out/ (developer tool).

usage: python tools/make_profile.py r01      (after tools/evidence.sh ran on the GPU box)
Copies the launch lists, the traversal DRAM CSV and the bench lines into profiles/, updates the measured
traversal traffic that bench.py reports, and writes the markdown summary (launch shares, DRAM traffic per
traversal launch, the round-2 --set full capture and its hottest source lines).
"""
import contextlib
import io
import json
import os
import runpy
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
T = os.path.join(ROOT, "tools")


def capture(script, *args):
    buf = io.StringIO()
    old = sys.argv
    sys.argv = [script, *args]
    try:
        with contextlib.redirect_stdout(buf):
            runpy.run_path(os.path.join(T, script), run_name="__main__")
    finally:
        sys.argv = old
    return buf.getvalue().rstrip()


def last_json(path):
    for line in reversed(open(path).read().strip().splitlines()):
        if line.startswith("{"):
            return json.loads(line)
    raise ValueError(path)


def main(tag):
    out = [f"# {tag} ncu evidence\n",
           "Produced by `tools/evidence.sh` on one B200 (`--clock-control none`) and summarised by "
           "`tools/make_profile.py`; raw CSVs sit next to this file, the bench lines in "
           f"`{tag}_bench.jsonl`. ncu serialises launches and starts cold, so absolute times differ slightly "
           "from `bench.py`; the *shares* are what matter.\n"]
    lines = []
    for f in ("bench_default.log", "bench_reference.log", "bench_blobs2d_24m.log", "bench_uniform2d_10m.log",
              "bench_normal3d_10m.log"):
        p = os.path.join(G, f)
        if os.path.exists(p):
            with contextlib.suppress(Exception):
                lines.append(last_json(p))
    if lines:
        with open(os.path.join(P, f"{tag}_bench.jsonl"), "w") as fh:
            for d in lines:
                fh.write(json.dumps(d) + "\n")
        out.append("| config | impl | MFeat/s | ms / solve | e2e MFeat/s | traversal ms | roofline frac (traversal) |")
        out.append("|---|---|---|---|---|---|---|")
        for d in lines:
            rf = d.get("roofline", {})
            out.append(f"| {d['config']['workload']} | {d.get('impl', 'ours')} | {d['value']:.1f} | {d['ms_per_step']:.2f} | "
                       f"{d['e2e']['value']:.1f} | {rf.get('ms_per_step', float('nan')):.2f} | {rf.get('frac', float('nan')):.3f} |")
        out.append("")
    for cfg in ("blobs3d_37m", "blobs2d_24m"):
        p = os.path.join(G, f"launches_{cfg}.csv")
        if os.path.exists(p):
            shutil.copy(p, os.path.join(P, f"{tag}_launches_{cfg}.csv"))
            out.append(f"## Step composition, {cfg} (`{tag}_launches_{cfg}.csv`)\n")
            out.append(capture("launch_summary.py", p))
            out.append("")
    traffic_path = os.path.join(P, f"{tag}_traverse_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {
        "note": "DRAM bytes of every k_traverse launch of one solve, from ncu --metrics dram__bytes_read.sum,"
                "dram__bytes_write.sum (tools/evidence_r02.sh); bench.py reports dram_bytes_per_launch as roofline.traffic"}
    for cfg in ("blobs3d_37m", "blobs2d_24m"):
        p = os.path.join(G, f"trav_dram_{cfg}.csv")
        if os.path.exists(p):
            shutil.copy(p, os.path.join(P, f"{tag}_trav_dram_{cfg}.csv"))
            txt = capture("trav_traffic.py", p)
            traffic[cfg] = json.loads(txt.splitlines()[-1])
            out.append(f"## Traversal DRAM traffic per launch, {cfg}\n\n```\n{txt}\n```\n")
    if traffic:
        with open(traffic_path, "w") as fh:
            json.dump(traffic, fh, indent=1)
    rep = os.path.join(G, "trav_r2_blobs3d_37m.ncu-rep")
    if os.path.exists(rep):
        out.append("## k_traverse, round 2 of blobs3d_37m, `--set full` (`trav_r2_blobs3d_37m.ncu-rep`, 8 MB, not committed)\n")
        out.append("| kernel | metric | value |\n|---|---|---|")
        out.append(capture("ncu_summary.py", rep))
        out.append("\nHottest source lines (stall samples, instructions, active threads per executed instruction):\n")
        out.append("```\n" + capture("line_hot.py", rep, "25") + "\n```\n")
        out.append("Reading: the traversal is bound by L2 latency and instruction issue, not by HBM bandwidth. "
                   "Issue slots are about half busy, about half the lanes of a warp are active, long-scoreboard "
                   "stalls sit on the packed box test that consumes the 64-byte node record, the L2 hit rate is "
                   "about 80 % and DRAM throughput is a few per cent. Its HBM roofline fraction is low by "
                   "construction: the algorithmic bytes (SURVEY §8d, 72 B per query per round in 3D) are re-read "
                   "from L2 about 25 times per round. The levers are fewer visits per query (tighter radii, "
                   "settling queries up front) and fewer instructions per visit (DESIGN.md §4).\n")
    with open(os.path.join(P, f"{tag}_profile.md"), "w") as fh:
        fh.write("\n".join(out) + "\n")
    print("wrote", os.path.join(P, f"{tag}_profile.md"))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
