"""Per-launch table of an ncu --metrics ...,dram__bytes_read.sum,dram__bytes_write.sum --csv
launch list: kernel, grid, duration (us), DRAM read+write (bytes)."""
import csv
import sys
from collections import OrderedDict

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "us": 1.0,
         "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def launches(path):
    with open(path) as f:
        rows = list(csv.reader(line for line in f if line.startswith('"')))
    hdr = rows[0]
    ii, ki, gi = hdr.index("ID"), hdr.index("Kernel Name"), hdr.index("Grid Size")
    ni, vi, ui = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    out = OrderedDict()
    for r in rows[1:]:
        d = out.setdefault(r[ii], {"kernel": r[ki].split("(")[0].replace("ibmg::", "").replace("void ", ""),
                                   "grid": r[gi]})
        d[r[ni]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
    return list(out.values())


if __name__ == "__main__":
    print(f"{'kernel':28s} {'grid':>16s} {'us':>10s} {'dram_bytes':>14s} {'GB/s':>8s}")
    for d in launches(sys.argv[1]):
        b = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        us = d.get("gpu__time_duration.sum", 0)
        print(f"{d['kernel'][:28]:28s} {d['grid']:>16s} {us:10.2f} {b:14.0f} {b / us / 1e3 if us else 0:8.1f}")
