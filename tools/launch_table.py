"""Per-kernel average durations from an ncu --csv launch list (gpu__time_duration.sum).
usage: python tools/launch_table.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(list)
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}
for r in rows[hi + 1:]:
    if len(r) > vi:
        agg[r[ki].split("(")[0][:48]].append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1))
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k:48s} n={len(v):3d} avg={sum(v) / len(v):9.1f} us")
