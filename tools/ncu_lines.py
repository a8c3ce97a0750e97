"""Summarise an ncu source page (--print-source cuda,sass --csv) per CUDA line:
stall samples and executed warp instructions (profiles/ summaries)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, x in enumerate(rows) if x and x[0] == "Line No")
h = rows[hi]
ni = h.index("# Samples")
ei = h.index("Instructions Executed")
line_rows = [x for x in rows[hi + 1:] if len(x) > ei and x[2] == "-"]   # cuda-line aggregate rows
tot_s = sum(float(x[ni] or 0) for x in line_rows) or 1
tot_e = sum(float(x[ei] or 0) for x in line_rows) or 1
print(f"total samples {tot_s:.0f}  executed warp instr {tot_e:.3e}")
line_rows.sort(key=lambda x: -float(x[ni] or 0))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for x in line_rows[:top]:
    print(f"{x[0]:>5s} {float(x[ni] or 0) / tot_s * 100:5.1f}%samp {float(x[ei] or 0) / tot_e * 100:5.1f}%inst | {x[1].strip()[:100]}")
