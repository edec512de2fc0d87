"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel launches, total/avg time and share (cold-cache, serialised)."""
import csv
import sys
from collections import defaultdict


def main(path):
    tot = defaultdict(lambda: [0, 0.0])
    with open(path) as f:
        rows = [r for r in csv.reader(line for line in f if line.startswith('"'))]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("ibmg::", "")
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3}.get(r[ui], 1e-3)
        tot[name][0] += 1
        tot[name][1] += v * scale
    all_us = sum(v[1] for v in tot.values())
    print(f"{'kernel':40s} {'launches':>9s} {'total_us':>12s} {'avg_us':>9s} {'share':>7s}")
    for k, (n, us) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:40s} {n:9d} {us:12.1f} {us / n:9.2f} {us / all_us:7.3f}")
    print(f"{'TOTAL':40s} {sum(v[0] for v in tot.values()):9d} {all_us:12.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
