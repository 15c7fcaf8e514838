"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel count, total, share."""
import collections
import csv
import sys


def summarise(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    agg = collections.OrderedDict()
    for r in data:
        name = r[ki].split("(")[0].replace("void ", "")[:48]
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    out = [f"{'kernel':48s} {'launches':>8s} {'total us':>12s} {'us/launch':>10s} {'share':>6s}"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:48s} {c:8d} {t:12.1f} {t / c:10.1f} {100 * t / tot:5.1f}%")
    out.append(f"{'TOTAL':48s} {sum(a[0] for a in agg.values()):8d} {tot:12.1f}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
