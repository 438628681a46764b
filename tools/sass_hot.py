"""Hot SASS lines of an ncu report (source page, sass view): stall samples, executions, active threads."""
import csv, subprocess, sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
idx = {k: h.index(k) for k in ["Address", "Source", "Warp Stall Sampling (All Samples)", "Instructions Executed",
                                "Avg. Threads Executed", "L2 Theoretical Sectors Local"]}
recs = []
for r in rows[2:]:
    try:
        recs.append((r[idx["Address"]], r[idx["Source"]], int(r[idx["Warp Stall Sampling (All Samples)"]] or 0),
                     int(r[idx["Instructions Executed"]] or 0), float(r[idx["Avg. Threads Executed"]] or 0),
                     int(r[idx["L2 Theoretical Sectors Local"]] or 0)))
    except (ValueError, IndexError):
        pass
tot_s = sum(x[2] for x in recs) or 1
tot_i = sum(x[3] for x in recs) or 1
print(f"{len(recs)} sass, samples {tot_s}, inst {tot_i:.3e}, thread-inst avg {sum(x[3]*x[4] for x in recs)/tot_i:.2f}")
print("local L2 sectors:", sum(x[5] for x in recs))
mode = sys.argv[3] if len(sys.argv) > 3 else "stall"
if mode == "all":
    for a, s, st, n, t, loc in recs:
        print(f"{a} {100*st/tot_s:5.1f}% {n:11d} {t:5.1f} {s[:90]}")
else:
    for a, s, st, n, t, loc in sorted(recs, key=lambda x: -x[2])[:top]:
        print(f"{a} {100*st/tot_s:5.1f}% {n:11d} {t:5.1f} {s[:90]}")
