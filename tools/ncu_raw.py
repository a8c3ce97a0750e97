"""Selected metrics from an ncu raw page (--page raw --csv)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
units = rows[1]
keys = sys.argv[2:] or ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
                        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
                        "launch__occupancy_limit_registers", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                        "dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
                        "launch__shared_mem_per_block_dynamic"]
for r in rows[2:]:
    for k in keys:
        if k in hdr:
            i = hdr.index(k)
            print(f"{k:70s} {r[i]:>20s} {units[i]}")
    st = [(float(r[i]) if r[i] else 0, h) for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")]
    tot = sum(v for v, _ in st) or 1
    for v, h in sorted(st, reverse=True)[:10]:
        print(f"  stall {h[len('smsp__pcsamp_warps_issue_stalled_'):]:40s} {v / tot:.3f}")
