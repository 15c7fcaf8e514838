"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ai, si, ci = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
ni = hdr.index("Warp Stall Sampling (Not-issued Samples)")
data = [r for r in rows[2:] if len(r) > ci and r[ci].strip()]
tot = sum(float(r[ci]) for r in data)
top = sorted(data, key=lambda r: -float(r[ci]))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]
for r in top:
    print(f"{r[ai]:>6s} {100 * float(r[ci]) / tot:5.1f}%  {r[si][:90]}")
