"""Tabulate ncu --csv metric dumps (one file per variant): rows = metrics, columns = variant/launch."""
import csv
import sys
from collections import OrderedDict

cols = OrderedDict()
for f in sys.argv[1:]:
    name = f.split("ncuvar_")[-1].replace(".csv", "")
    lines = open(f).read().splitlines()
    i = next(j for j, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[i:]))
    h = rows[0]
    iid, im, iv = h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
    for r in rows[1:]:
        key = f"{name}:{r[iid]}"
        cols.setdefault(key, OrderedDict())[r[im]] = r[iv]
metrics = list(next(iter(cols.values())).keys())
w = max(len(m) for m in metrics)
print(" " * w, *[f"{k:>16s}" for k in cols])
for m in metrics:
    print(f"{m:{w}s}", *[f"{cols[k].get(m, ''):>16s}" for k in cols])
