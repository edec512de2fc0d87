"""Condense an `ncu -i X.ncu-rep --page details --csv` export into the key
lines (speed of light, occupancy, scheduler and warp-state statistics)."""
import csv
import sys

KEEP = ["Memory Throughput", "DRAM Throughput", "Duration", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Issue Slots Busy", "Mem Busy", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Active Warps Per Scheduler", "Eligible Warps Per Scheduler", "No Eligible", "Warp Cycles Per Issued Instruction",
        "Grid Size", "Block Size", "Registers Per Thread", "Dynamic Shared Memory Per Block", "Block Limit Registers",
        "Block Limit Shared Mem", "Theoretical Occupancy", "Achieved Occupancy", "Executed Ipc Active"]


def main(path):
    with open(path) as f:
        rows = list(csv.reader(line for line in f if line.startswith('"')))
    hdr = rows[0]
    si, ni, ui, vi = (hdr.index(k) for k in ("Section Name", "Metric Name", "Metric Unit", "Metric Value"))
    seen = set()
    print(rows[1][hdr.index("Kernel Name")])
    for r in rows[1:]:
        if r[ni] in KEEP and r[ni] not in seen:
            seen.add(r[ni])
            print(f"{r[si][:28]:28s} {r[ni]:45s} {r[vi]:>12s} {r[ui]}")


if __name__ == "__main__":
    main(sys.argv[1])
