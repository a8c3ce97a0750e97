"""Summarise one ncu --set full report: key raw metrics, stall mix, instruction mix per family.
usage: python tools/ncu_summary.py REPORT.ncu-rep FAMILIES [hot-sass-out.txt]"""
import csv
import collections
import io
import subprocess
import sys

rep, fams = sys.argv[1], float(sys.argv[2])


def page(args):
    out = subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


rows = page(["--page", "raw", "--csv"])
h = rows[0]
# several launches captured: summarise the longest one
ti = h.index("gpu__time_duration.sum")
best = max(range(2, len(rows)), key=lambda r: float(rows[r][ti] or 0))
d = dict(zip(h, rows[best]))
launch_id = d.get("ID")
for k in ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
          "dram__bytes_write.sum", "dram__bytes_read.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
          "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
          "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
          "launch__shared_mem_per_block_dynamic", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]:
    print(f"  {k:70s} {d.get(k)}")
rows = page(["--page", "source", "--csv", "--print-source", "sass"])
heads = [i for i, x in enumerate(rows) if x and x[0] == "Address"]
def section(k):
    h = rows[heads[k]]
    end = heads[k + 1] if k + 1 < len(heads) else len(rows)
    return h, [x for x in rows[heads[k] + 1:end] if len(x) == len(h)]


def weight(k):
    h, data = section(k)
    ei = h.index("Instructions Executed")
    return sum(float(x[ei] or 0) for x in data)


h, data = section(max(range(len(heads)), key=weight))   # the launch with the most instructions
si, ei = h.index("Source"), h.index("Instructions Executed")
sc = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
tot = collections.Counter()
op = collections.Counter()
for x in data:
    for i in sc:
        tot[h[i]] += float(x[i] or 0)
    s = x[si].strip()
    if s:
        o = s.split()[0]
        if o.startswith("@"):
            o = s.split()[1]
        op[o.split(".")[0]] += float(x[ei] or 0)
T = sum(tot.values()) or 1
print("stalls:", " ".join(f"{k[6:]}:{100 * v / T:.1f}" for k, v in tot.most_common(8)))
ti = sum(op.values())
print(f"warp inst/family {ti / fams:.3f}:", " ".join(f"{o}:{c / fams:.3f}" for o, c in op.most_common(24)))
if len(sys.argv) > 3:
    vals = [float(x[ei] or 0) for x in data]
    mx = max(vals)
    with open(sys.argv[3], "w") as f:
        for i, x in enumerate(data):
            if vals[i] >= 0.1 * mx:
                f.write(f"{i:5d} {vals[i] / mx:6.3f} {x[si].strip()[:100]}\n")

if len(sys.argv) > 4:
    # basic blocks (runs of equal execution count) by instruction share
    si, ei = h.index("Source"), h.index("Instructions Executed")
    vals = [float(x[ei] or 0) for x in data]
    tot = sum(vals) or 1
    blocks, start = [], 0
    for i in range(1, len(vals) + 1):
        if i == len(vals) or vals[i] != vals[start]:
            blocks.append((start, i, vals[start] * (i - start), vals[start]))
            start = i
    blocks.sort(key=lambda b: -b[2])
    acc = 0
    for b in blocks[:int(sys.argv[4])]:
        acc += b[2]
        ops = collections.Counter(data[j][si].strip().split()[0].lstrip("@!P0123456789T ").split(".")[0]
                                  if not data[j][si].strip().startswith("@") else data[j][si].strip().split()[1].split(".")[0]
                                  for j in range(b[0], b[1]))
        print(f"{b[0]:5d}-{b[1]:5d} n={b[1] - b[0]:3d} cnt={b[3]:.3e} share={100 * b[2] / tot:5.2f}% cum={100 * acc / tot:5.1f}% "
              + " ".join(f"{o}:{c}" for o, c in ops.most_common(6)))
