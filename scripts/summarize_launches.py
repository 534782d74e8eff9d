"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list: per-kernel launches, total
device time and share.  Usage: python scripts/summarize_launches.py launches.csv"""
import collections
import csv
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= mi:
        continue
    name = r[ki].split("(")[0]
    v = float(r[mi].replace(",", "")) * SCALE[r[ui]]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
print(f"{sum(a[0] for a in agg.values())} launches, total {tot:.1f} ms (ncu: serialised, cold-cache)")
print(f"{'ms':>10} {'share':>6} {'n':>5}  kernel")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t:10.2f} {100 * t / tot:5.1f}% {c:5d}  {k}")
