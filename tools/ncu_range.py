"""Print a range of an ncu SASS source page (--print-source sass --csv): index, executed warp
instructions, stall samples, instruction text."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, x in enumerate(rows) if x and x[0] == "Address")
h = rows[hi]
data = rows[hi + 1:]
si = h.index("Source")
ni = h.index("Warp Stall Sampling (All Samples)")
ei = h.index("Instructions Executed")
a, b = int(sys.argv[2]), int(sys.argv[3])
minexec = float(sys.argv[4]) if len(sys.argv) > 4 else 0
for i in range(a, min(b, len(data))):
    x = data[i]
    e = float(x[ei] or 0)
    if e < minexec:
        continue
    print(f"{i:5d} {e:12.0f} {float(x[ni] or 0):7.0f}  {x[si].strip()[:90]}")
