"""Per-CUDA-line instruction counts and stall samples from an ncu report (cuda,sass view)."""
import csv, subprocess, sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname = None
recs = []
hdr = None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        st = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        n = int(r[hdr.index("Instructions Executed")])
        t = int(r[hdr.index("Thread Instructions Executed")])
    except ValueError:
        continue
    recs.append((fname, r[0], r[1], st, n, t))
ts = sum(x[3] for x in recs) or 1
ti = sum(x[4] for x in recs) or 1
print(f"warp inst {ti:.3e}  thread/warp {sum(x[5] for x in recs)/ti:.2f}")
key = 4 if (len(sys.argv) > 3 and sys.argv[3] == "inst") else 3
for f, ln, src, st, n, t in sorted(recs, key=lambda x: -x[key])[:top]:
    print(f"{f}:{ln:>4} stall {100*st/ts:5.1f}% inst {100*n/ti:5.1f}% thr {t/max(n,1):5.1f} | {src.strip()[:80]}")
