"""Summarise an ncu report (details page) into the metrics we track; usage: ncu_summary.py report.ncu-rep"""
import csv, subprocess, sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Compute (SM) Throughput", "Issue Slots Busy", "Executed Ipc Active", "Avg. Active Threads Per Warp",
        "Avg. Not Predicated Off Threads Per Warp", "Achieved Occupancy", "Theoretical Occupancy",
        "Registers Per Thread", "Executed Instructions", "Branch Efficiency", "Warp Cycles Per Issued Instruction",
        "Eligible Warps Per Scheduler", "No Eligible", "Grid Size", "Block Size", "Local Memory Spilling Requests"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    ki, mi, ui, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    seen = set()
    for r in rows[1:]:
        if r[mi] in KEYS and (r[ki], r[mi]) not in seen:
            seen.add((r[ki], r[mi]))
            print(f"| {r[ki][:40]} | {r[mi]} | {r[vi]} {r[ui]} |")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if len(rr) > 2:
        hdr, units, vals = rr[0], rr[1], rr[2:]
        want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
                "smsp__thread_inst_executed_per_inst_executed.ratio",
                "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_imc_miss_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_drain_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_tex_throttle_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio"]
        for v in vals:
            for w in want:
                if w in hdr:
                    i = hdr.index(w)
                    print(f"| {v[hdr.index('Kernel Name')][:40]} | {w} | {v[i]} {units[i]} |")


if __name__ == "__main__":
    main(sys.argv[1])
