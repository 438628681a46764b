"""DRAM traffic of every traversal launch from an ncu metrics CSV (developer tool).

usage: trav_traffic.py trav_dram_<cfg>.csv  ->  per-launch GB / ms and the per-launch mean (JSON on the last line)
"""
import csv, json, sys

BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
SECS = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def main(path):
    rows = [r for r in csv.reader(open(path)) if r]
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    mi, vi, ui, iid = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit"), hdr.index("ID")
    per = {}
    for r in rows[h + 1:]:
        per.setdefault(r[iid], {})[r[mi]] = (float(r[vi].replace(",", "")), r[ui])
    launches = []
    for k, v in per.items():
        rb, wb, t = v["dram__bytes_read.sum"], v["dram__bytes_write.sum"], v["gpu__time_duration.sum"]
        b = rb[0] * BYTES[rb[1]] + wb[0] * BYTES[wb[1]]
        s = t[0] * SECS[t[1]]
        launches.append((b, s))
        print(f"launch {k}: {b / 1e9:.3f} GB in {s * 1e3:.3f} ms")
    tb = sum(b for b, _ in launches)
    ts = sum(s for _, s in launches)
    print(json.dumps({"launches": len(launches), "dram_bytes_total": tb, "dram_bytes_per_launch": tb / len(launches),
                      "ncu_ms_total": ts * 1e3}))


if __name__ == "__main__":
    main(sys.argv[1])
