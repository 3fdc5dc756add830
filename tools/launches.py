"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[h], rows[h + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}
    out = []
    for r in data:
        out.append((r[ki], float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)))
    return out


if __name__ == "__main__":
    L = load(sys.argv[1])
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = sum(t for _, t in L)
    for name, t in L:
        k = name.split("(")[0]
        agg[k][0] += 1
        agg[k][1] += t
    print(f"{'kernel':58s} {'n':>5s} {'total_us':>10s} {'avg_us':>8s} share")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:58]:58s} {n:5d} {t / 1e3:10.1f} {t / n / 1e3:8.2f} {t / tot:.3f}")
    if len(sys.argv) > 2:
        top = sorted(L, key=lambda x: -x[1])[: int(sys.argv[2])]
        for name, t in top:
            print(f"  {t / 1e3:9.1f} us  {name[:100]}")
