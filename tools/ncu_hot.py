"""Top SASS instructions by warp-stall samples from `ncu --page source --csv`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
si, ai, ni = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
body = [r for r in rows[2:] if len(r) > ai and r[ai].replace(".", "", 1).isdigit()]
tot = sum(float(r[ai] or 0) for r in body)
top = sorted(body, key=lambda r: -float(r[ai] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]
print(f"total samples {tot:.0f}, instructions {len(body)}")
for r in top:
    print(f"{float(r[ai]):7.0f} {100 * float(r[ai]) / tot:5.1f}%  {r[si].strip()[:90]}")
