"""Summarise an ncu launch list (gpu__time_duration.sum CSV): per-kernel totals and share of the step."""
import csv, collections, sys


def load(path):
    rows = [r for r in csv.reader(open(path)) if r]
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    out = []
    for r in rows[h + 1:]:
        v = float(r[vi].replace(",", ""))
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}[r[ui]]
        out.append((r[ki], v * scale))
    return out


def short(name):
    name = name.split("(")[0]
    return name.replace("void ", "").replace("emst::", "")


def main(path, top=25):
    launches = load(path)
    total = sum(t for _, t in launches)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k, t in launches:
        a = agg[short(k)]
        a[0] += 1
        a[1] += t
    print(f"{len(launches)} launches, {total:.3f} ms summed (serialised, ncu)")
    print("| kernel | launches | ms | share |\n|---|---|---|---|")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"| `{k}` | {c} | {t:.3f} | {100 * t / total:.1f} % |")


if __name__ == "__main__":
    main(sys.argv[1])
