"""Summarise ncu outputs (launch list CSV + one --set full capture) into profiles/.

usage: python tools/summarize_profiles.py <launches.csv> <prof.ncu-rep> <config> <tag>
Writes profiles/<tag>_launches.md and profiles/<tag>_walk_ncu.md, and
profiles/traverse_ncu_summary.json (read by bench.py for roofline.traffic).
The capture holds the walk kernel's launches of one step (one per shared-memory
class): their DRAM bytes are summed (the bench's "dominant kernel" is all of
them, timed together)."""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
launches, rep, config, tag = sys.argv[1:5]
out = os.path.join(ROOT, "profiles")


def to_ns(v, u):
    v = float(v.replace(",", ""))
    return v * {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(u, 1)


rows = list(csv.reader(open(launches)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("void ", "").replace("bnr::", "")
    name = name.split("<")[0]
    agg[name][0] += 1
    agg[name][1] += to_ns(r[vi], r[ui])
tot = sum(a[1] for a in agg.values())
lines = [f"# {tag}: kernel launch list ({config})", "",
         "`ncu --metrics gpu__time_duration.sum --clock-control none` over `python bench.py --no-e2e "
         "--no-cpu-baseline --steps 2 --warmup 1` (cold-cache, serialised launches: compare shares).", "",
         "| kernel | launches | total ms | avg us | share |", "|---|---|---|---|---|"]
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    lines.append(f"| {k} | {c} | {t / 1e6:.3f} | {t / c / 1e3:.1f} | {t / tot:.3f} |")
open(os.path.join(out, f"{tag}_launches.md"), "w").write("\n".join(lines) + "\n")

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
names, units = r[0], r[1]
launch_rows = r[2:]


def val(row, k):
    i = names.index(k)
    return float(row[i].replace(",", "") or 0), units[i]


def to_bytes(v, u):
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)


keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
        "launch__grid_size", "launch__shared_mem_per_block_dynamic",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "lts__t_sectors_op_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
md = [f"# {tag}: walk_kernel, ncu --set full ({config})", "",
      f"The walk kernel's {len(launch_rows)} launch(es) of one step (one per shared-memory class), "
      "`ncu --set full --clock-control none --import-source on`.", "",
      "| metric | " + " | ".join(f"launch {j}" for j in range(len(launch_rows))) + " |",
      "|---|" + "---|" * len(launch_rows)]
for k in keys:
    if k in names:
        md.append(f"| {k} | " + " | ".join(f"{row[names.index(k)]} {units[names.index(k)]}" for row in launch_rows) + " |")
# stall mix of the longest launch
ti = names.index("gpu__time_duration.sum")
big = max(launch_rows, key=lambda row: float(row[ti].replace(",", "") or 0))
stall = [k for k in names if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")]
sv = sorted(((float(big[names.index(k)].replace(",", "") or 0), k) for k in stall), reverse=True)
st = sum(x for x, _ in sv) or 1
md += ["", "| stall reason (pc sampling, longest launch) | share |", "|---|---|"]
for x, k in sv[:10]:
    md.append(f"| {k.replace('smsp__pcsamp_warps_issue_stalled_', '')} | {x / st:.3f} |")
open(os.path.join(out, f"{tag}_walk_ncu.md"), "w").write("\n".join(md) + "\n")

rd = sum(to_bytes(*val(row, "dram__bytes_read.sum")) for row in launch_rows)
wr = sum(to_bytes(*val(row, "dram__bytes_write.sum")) for row in launch_rows)
summary = {"config": config, "tag": tag, "kernel": "walk_kernel", "launches_per_step": len(launch_rows),
           "traffic_bytes_per_launch": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
           "note": "per step: the sum over the walk kernel's per-class launches"}
json.dump(summary, open(os.path.join(out, "traverse_ncu_summary.json"), "w"), indent=1)
print(open(os.path.join(out, f"{tag}_launches.md")).read())
print(open(os.path.join(out, f"{tag}_walk_ncu.md")).read())
