"""Top SASS instructions for one stall reason of an ncu SASS source page."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, x in enumerate(rows) if x and x[0] == "Address")
h = rows[hi]
d = rows[hi + 1:]
si = h.index("Source")
li = h.index("stall_" + sys.argv[2])
tot = sum(float(x[li] or 0) for x in d) or 1
alls = sum(float(x[h.index("Warp Stall Sampling (All Samples)")] or 0) for x in d)
print(f"{sys.argv[2]}: {tot / alls * 100:.1f}% of all samples")
for i in sorted(range(len(d)), key=lambda i: -float(d[i][li] or 0))[: int(sys.argv[3]) if len(sys.argv) > 3 else 20]:
    print(f"{i:5d} {float(d[i][li] or 0) / tot * 100:5.1f}% {d[i][si][:60]:60s} | prev: {d[i - 1][si][:45]}")
