"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per kernel name,
launches, total and mean duration, share of the total (dev tool; profiles/*_launches_summary.txt)."""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    acc = defaultdict(list)
    for r in rows[start + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            name = r[ki].split("(")[0]
            acc[name].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in acc.values()) or 1.0
    print(f"{'kernel':60s} {'launches':>8s} {'total_us':>10s} {'mean_us':>9s} {'share':>6s}")
    for k, v in sorted(acc.items(), key=lambda kv: -sum(kv[1])):
        s = sum(v)
        print(f"{k[:60]:60s} {len(v):8d} {s / 1e3:10.1f} {s / len(v) / 1e3:9.2f} {100 * s / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
