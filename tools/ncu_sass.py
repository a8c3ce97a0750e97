"""Top SASS instructions of an ncu source page (--print-source sass --csv) with stall reasons."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, x in enumerate(rows) if x and x[0] == "Address")
h = rows[hi]
data = rows[hi + 1:]
si = h.index("Source")
ni = h.index("Warp Stall Sampling (All Samples)")
ei = h.index("Instructions Executed")
sc = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(float(x[ni] or 0) for x in data) or 1
idx = sorted(range(len(data)), key=lambda i: -float(data[i][ni] or 0))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
for i in idx[:top]:
    x = data[i]
    reasons = sorted(((float(x[c] or 0), h[c][6:]) for c in sc), reverse=True)[:3]
    rs = " ".join(f"{n}:{v / tot * 100:.1f}" for v, n in reasons if v > 0)
    print(f"{i:5d} {float(x[ni] or 0) / tot * 100:5.1f}% {x[si].strip()[:60]:60s} {rs}")
    for j in range(max(0, i - ctx), i):
        print(f"        ctx {data[j][si].strip()[:70]}")
