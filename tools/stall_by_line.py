"""Warp-stall samples aggregated by CUDA source line, from
`ncu -i X.ncu-rep --page source --csv --print-source cuda,sass`."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
fname, agg, reasons = None, collections.Counter(), collections.defaultdict(collections.Counter)
src = {}
hdr = None
cur_line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5:
        continue
    if r[0].strip():
        cur_line = (fname, int(r[0]))
        src[cur_line] = r[1].strip()
    try:
        s = float(r[4] or 0)
    except ValueError:
        continue
    if cur_line and s:
        agg[cur_line] += s
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    reasons[cur_line][h[6:]] += float(r[i] or 0)
                except ValueError:
                    pass
tot = sum(agg.values())
for k, v in agg.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    top = ", ".join(f"{n} {100 * c / v:.0f}%" for n, c in reasons[k].most_common(3))
    print(f"{k[0]}:{k[1]:<5} {100 * v / tot:5.1f}%  [{top}]  {src.get(k, '')[:70]}")
