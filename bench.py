#!/usr/bin/env python
"""bench.py -- families (child, parent-set) RSS+BIC per second on B200.

One "step" = the whole hot path over one synthetic dataset: centre + TSQR of X
(a1-a2), [multi-GPU: NCCL broadcast of R (a3)], seed tree + fused traversal
(a4-a10: GRCs, suffix-sum harvest, BIC, RSS+BIC stores into the (child, mask)
table) + per-child best (a11) [multi-GPU: NCCL all-gather of the per-rank bests
and the deterministic merge].  Workload: BASELINE.json configs[4] (m=28,
n=2000; the config the north-star metric is quoted on; it fits one B200: the
RSS+BIC tables are 60 GB).

  python bench.py [--gpus N --steps K --warmup W] [--config C] [--impl reference]

Prints ONE JSON line on rank 0.  value = all families of all ranks / the max
over ranks of the device time of K steps (CUDA events on the launching stream,
barrier + synchronize on both sides).  e2e = the same metric through the
public C-ABI with X in pinned HOST memory (H2D inside the step) and the
per-child best read back to the host (D2H) every step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "families (child,parent-set) RSS+BIC per second"
UNIT = "families/s"
BYTES_PER_FAMILY = 16  # 8 B RSS + 8 B BIC written per family


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--seed", type=int, default=None)
    ap.add_argument("--k", type=int, default=0, help="free block size (0 = library default)")
    ap.add_argument("--lw", type=int, default=-1, help="seed-tree levels derived in-warp (-1 = default)")
    ap.add_argument("--pack-bits", type=int, default=0, help="log2 lockstep workers per warp (0 = library default)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--layout", default="pairs", choices=["pairs", "tables"],
                    help="pairs: one table of 16 B (RSS, BIC) records (bnreg_run_pairs, the north star's "
                         "128-bit stores); tables: separate RSS and BIC tables (bnreg_run)")
    ap.add_argument("--outputs", default="both", choices=["both", "rss", "bic", "none"],
                    help="diagnostic: which tables the timed run writes (the metric needs both)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sim-world", type=int, default=1,
                    help="diagnostic (one GPU, no collectives): run logical rank --sim-rank of a world of this size "
                         "(its shard of the lattice, rank-filtered seed tree) to measure per-rank costs")
    ap.add_argument("--sim-rank", type=int, default=0)
    ap.add_argument("--e2e-first", action="store_true",
                    help="diagnostic: time the e2e steps before the device-resident steps")
    ap.add_argument("--no-pipeline", action="store_true",
                    help="load each dataset on the walk's stream (no overlap of dataset s+1's load and seed "
                         "tree with dataset s's walk)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(cfg):
    """dram read+write bytes of the walk launches of one step, from the committed ncu
    capture (a capture value, not measured in this run): (bytes, source tag) or (None, None)."""
    p = os.path.join(ROOT, "profiles", "traverse_ncu_summary.json")
    if os.path.exists(p):
        d = json.load(open(p))
        if d.get("config") == cfg and d.get("traffic_bytes_per_launch"):
            return float(d["traffic_bytes_per_launch"]), "ncu --set full capture %s (profiles/traverse_ncu_summary.json)" % (
                d.get("tag"),)
    return None, None


# Measured on this pool's B200 (tools/microbench.cu, profiles/r01_microbench_b200.txt): the FP64 FMA
# peak and the store-only bandwidth of coalesced 16 B stores (the copy peak of MEASURED_PEAKS.json
# counts reads and writes)
FP64_PEAK_TFLOPS = 34.79
STORE_PEAK_GBS = 6967.5


def eq13_flops(m):
    """Eq.13 (reading G6): the Givens flops of the whole walk,
    3m 2^m + 6 2^m - 3m^2 - 9m - 6 (the roofline's FP64 term, north star)."""
    return 3 * m * 2 ** m + 6 * 2 ** m - 3 * m * m - 9 * m - 6


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None
        self.f = None

    def start(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.flush()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                for nm, val in zip(names, r[5:9]):
                    if val.strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------- oracle timing
def oracle_rate(X, seconds, seed=1234, batch=256):
    """The oracle (O1, per-family Householder, OpenMP over families) as it stands,
    on a bounded uniform sample of the workload's families; and the reduced oracle O2
    (Householder on slices of the oracle's root QR) on 1e6 sampled families."""
    import numpy as np
    import oracle
    n, m = X.shape
    Xc = oracle.centre(X)
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.integers(0, m << (m - 1), size=2_000_000)).astype(np.int64)
    done, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < seconds and done < len(idx):
        oracle.rss_indices(Xc, idx[done:done + batch])
        done += min(batch, len(idx) - done)
        batch = min(batch * 2, 8192)
    el = time.perf_counter() - t0
    t1 = time.perf_counter()
    R0 = oracle.qr_r(Xc)
    oracle.rss_reduced_indices(R0, idx[:1_000_000])
    o2 = 1_000_000 / (time.perf_counter() - t1)
    return done / el, done, el, oracle.num_threads(), o2


def bench_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import datagen
    X = datagen.config_data(args.config, args.seed)
    n, m = X.shape
    import numpy as np
    import oracle
    Xc = oracle.centre(X)
    per_step = 2048
    idx = datagen.sample_indices(m, per_step * (args.steps + args.warmup), 99)
    for s in range(args.warmup):
        oracle.rss_indices(Xc, idx[s * per_step:(s + 1) * per_step])
    t0 = time.perf_counter()
    for s in range(args.warmup, args.warmup + args.steps):
        r = oracle.rss_indices(Xc, idx[s * per_step:(s + 1) * per_step])
        _, S = oracle.masks_of(m, idx[s * per_step:(s + 1) * per_step])
        oracle.bic_array(r, n, [bin(int(q)).count("1") for q in S])
    el = time.perf_counter() - t0
    val = per_step * args.steps / el
    sample = (f"{per_step} families per step, uniform over the m*2^(m-1) = {m << (m - 1)} families "
              f"of cfg{args.config} (O1 per-family Householder QR + BIC, n={n})")
    out = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": {"workload": f"cfg{args.config}", "m": m, "n": n},
           "cpu_baseline": {"value": val, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------------------- ours
class NcclComm:
    """The step's two exchanges over torch.distributed on the current stream (NCCL over
    NVLink): a3 broadcast of the root R, a11 all-gather of the per-rank best records."""

    def __init__(self, dist):
        self.dist = dist

    def broadcast(self, t, src):
        self.dist.broadcast(t, src)

    def all_gather(self, out, t):
        self.dist.all_gather_into_tensor(out, t)


class HostStagedComm(NcclComm):
    """The same exchanges for a CPU-only backend (gloo): the device tensors are staged
    through host memory.  Used by the multi-process test on one GPU (tests/), where
    NCCL cannot put two ranks on one device."""

    def broadcast(self, t, src):
        c = t.cpu()
        self.dist.broadcast(c, src)
        t.copy_(c)

    def all_gather(self, out, t):
        import torch
        c = torch.empty(out.numel(), dtype=out.dtype)        # gloo wants a flat output
        self.dist.all_gather_into_tensor(c, t.cpu().reshape(-1))
        out.copy_(c.view(out.shape))


class Pipeline:
    """One bench step on this rank, through the C-ABI (paper_1901_07643_b200):
      rank 0: a1-a2 load (centre + TSQR) of X          [bnreg_load_async]
      N > 1:  a3 broadcast of R from rank 0              [bnreg_get/set_root_device + comm]
      every rank: a4-a11 seeds, walk, stores, best      [bnreg_run_pairs_async / bnreg_run_async]
      N > 1:  all-gather of the per-rank best records, device merge (G14)
                                                         [comm + bnreg_best_merge_async]
    No host synchronisation inside a device step; load errors surface at sync()."""

    def __init__(self, bn, h, X, world, rank, dev, comm=None, pairs=True, outputs="both", load_stream=None):
        import numpy as np
        import torch
        self.bn, self.h, self.world, self.rank, self.comm = bn, h, world, rank, comm
        # pipelined datasets: the load (and the R broadcast) of the next dataset on load_stream
        # while the current one is walked (bnreg_set_load_stream)
        self.load_stream = load_stream
        if load_stream is not None:
            h.set_load_stream(load_stream.cuda_stream)
        n, m = X.shape
        self.m = m
        F = h.num_families()
        self.pairs = pairs
        if pairs:
            self.tab = torch.empty((F, 2), dtype=torch.float64, device=dev)
            self.rss = self.bic = None
        else:
            self.tab = None
            self.rss = torch.empty(F, dtype=torch.float64, device=dev) if outputs in ("both", "rss") else None
            self.bic = torch.empty(F, dtype=torch.float64, device=dev) if outputs in ("both", "bic") else None
        self.Xd = torch.from_numpy(np.ascontiguousarray(X.T)).to(dev)          # column-major n x m
        self.Xpin = torch.from_numpy(np.ascontiguousarray(X.T)).pin_memory()
        self.Xpin_np = self.Xpin.numpy().T                                   # Fortran view of pinned memory
        self.Rt = torch.empty(m * m, dtype=torch.float64, device=dev)
        # this rank's best as one record [m BICs | m masks | pad] (16 m bytes): one all-gather
        self.rec = torch.empty(2 * m, dtype=torch.float64, device=dev)
        self.gat = torch.empty((world, 2 * m), dtype=torch.float64, device=dev)
        self.best_bic = torch.empty(m, dtype=torch.float64, device=dev)
        self.best_mask = torch.empty(m, dtype=torch.int32, device=dev)

    def _rec_ptrs(self, base):
        return base + 8 * self.m, base        # (masks, bics)

    def _exchange_root(self):
        if self.world > 1:
            import contextlib
            import torch
            ctx = torch.cuda.stream(self.load_stream) if self.load_stream is not None else contextlib.nullcontext()
            with ctx:
                if self.rank == 0:
                    self.h.get_root_device(self.Rt)
                self.comm.broadcast(self.Rt, 0)
                if self.rank != 0:
                    self.h.set_root_device(self.Rt)

    def _walk(self):
        bm, bb = self._rec_ptrs(self.rec.data_ptr())
        if self.world == 1:
            bm, bb = self.best_mask.data_ptr(), self.best_bic.data_ptr()
        if self.pairs:
            self.h.run_pairs_async(self.tab, bm, bb)
        else:
            self.h.run_async(self.rss, self.bic, bm, bb)

    def _merge(self):
        if self.world > 1:
            self.comm.all_gather(self.gat, self.rec)
            gm, gb = self._rec_ptrs(self.gat.data_ptr())
            self.h.best_merge_async(self.world, gm, gb, self.best_mask, self.best_bic, row_bytes=16 * self.m)

    def step_device(self):
        """Inputs resident in HBM."""
        if self.rank == 0:
            self.h.load_async(self.Xd)
        self._exchange_root()
        self._walk()
        self._merge()

    def step_e2e(self):
        """X from pinned host memory (H2D inside the step), the merged per-child best read
        back to the host (D2H) -- returns (best_mask, best_bic) numpy.  Pipelined (a load
        stream): the D2H goes asynchronously into pinned memory and the host reads the
        previous step's result, so step s+1's upload and prep overlap step s; every step's
        result is still copied to and read on the host (the last one by finish_e2e)."""
        import numpy as np
        import torch
        if self.rank == 0:
            self.h.load_async(self.Xpin_np)
        self._exchange_root()
        self._walk()
        self._merge()
        if self.load_stream is None:
            bm = self.best_mask.cpu().numpy().view(np.uint32)
            bb = self.best_bic.cpu().numpy()
            return bm, bb
        if not hasattr(self, "_hbest"):
            self._hbest = [(torch.empty(self.m, dtype=torch.int32).pin_memory(),
                            torch.empty(self.m, dtype=torch.float64).pin_memory()) for _ in range(2)]
            self._hev = [torch.cuda.Event(), torch.cuda.Event()]
            self._slot = 0
            self._pending = None
        s = self._slot
        self._hbest[s][0].copy_(self.best_mask, non_blocking=True)
        self._hbest[s][1].copy_(self.best_bic, non_blocking=True)
        self._hev[s].record()
        prev, self._pending, self._slot = self._pending, s, 1 - s
        if prev is None:
            return None
        return self._read_host(prev)

    def _read_host(self, s):
        import numpy as np
        self._hev[s].synchronize()
        return self._hbest[s][0].numpy().view(np.uint32).copy(), self._hbest[s][1].numpy().copy()

    def finish_e2e(self):
        """The last pipelined step's result (None without pipelining)."""
        if getattr(self, "_pending", None) is None:
            return None
        r = self._read_host(self._pending)
        self._pending = None
        return r

    def h2d_bytes(self):
        return self.Xd.numel() * 8 if self.rank == 0 else 0

    def d2h_bytes(self):
        return self.m * (4 + 8)


def bench_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    import datagen
    import paper_1901_07643_b200 as bn

    world, rank, local = dist_env()
    if world != args.gpus:
        args.gpus = world
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    X = datagen.config_data(args.config, args.seed)
    n, m = X.shape
    sim = args.sim_world > 1 and world == 1
    opt = bn.options(free_vars=args.k, levels_in_warp=args.lw, world=args.sim_world if sim else world,
                     rank=args.sim_rank if sim else rank, pack_bits=args.pack_bits)
    h = bn.Bnreg(n, m, opt)
    plan = bn.bnreg_plan_query(m, n, opt)
    # one explicit (non-legacy) stream for torch, NCCL ordering and the handle: the timing
    # events are recorded on the stream the kernels run on
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    h.set_stream(stream.cuda_stream)
    F = h.num_families()
    total = m << (m - 1)
    pairs = args.layout == "pairs" and args.outputs == "both"
    load_stream = None if args.no_pipeline else torch.cuda.Stream(dev)
    pipe = Pipeline(bn, h, X, world, rank, dev, NcclComm(dist) if world > 1 else None, pairs, args.outputs,
                    load_stream)
    step_device, step_e2e = pipe.step_device, pipe.step_e2e

    def timed(step, k, w, with_clocks=False):
        for _ in range(w):
            step()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        clk = Clocks(local) if with_clocks else None
        if clk:
            clk.start()
            time.sleep(0.3)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        if load_stream is not None:
            load_stream.wait_event(e0)          # every timed load starts after e0
        for _ in range(k):
            step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        ms = e0.elapsed_time(e1)
        clocks = clk.stop() if clk else None
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, clocks

    # device-resident inputs: the headline value (no host synchronisation inside the timed
    # steps), then the same steps again with the handle's per-phase CUDA events (the
    # traversal kernel's own time; collecting them synchronises once per step)
    h.timing(0)
    if args.e2e_first and not args.no_e2e:
        ms_e2e_first, clocks_e2e = timed(step_e2e, args.steps, args.warmup, with_clocks=True)
        pipe.finish_e2e()
    ms, clocks = timed(step_device, args.steps, args.warmup, with_clocks=True)
    h.sync()                                   # deferred load checks (NaN/Inf, rank)
    h.timing(1)
    ms_chk, _ = timed(step_device, args.steps, 0)
    tms, runs = h.timing(0)
    trav_ms = tms[2] / max(runs, 1)
    run_ms = tms[0] / max(runs, 1)
    phases = {"load_ms (rank 0: centre + root QR)": (tms[4] / tms[5]) if tms[5] else None,
              "seeds_ms (seed tree + seed kernel)": tms[1] / max(runs, 1), "walk_ms": trav_ms,
              "best_reduce_ms": tms[3] / max(runs, 1), "run_ms (seeds + walk + reduce)": run_ms}
    value = (F if sim else total) * args.steps / (ms / 1e3)
    e2e = None
    if not args.no_e2e:
        # the same protocol as the device-resident steps (warm-up, then the clock sampler's
        # 0.3 s start before the timed region), so both numbers start from the same GPU state
        if args.e2e_first:
            ms_e2e = ms_e2e_first
        else:
            ms_e2e, clocks_e2e = timed(step_e2e, args.steps, args.warmup, with_clocks=True)
            pipe.finish_e2e()
        e2e = {"value": total * args.steps / (ms_e2e / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": n * m * 8, "d2h_bytes_per_step": world * pipe.d2h_bytes(),
               "pipelined": ("each step's best is copied asynchronously to pinned host memory and read on the "
                             "host one step later (the last after the timed loop's synchronisation)"
                             if load_stream is not None else "no"),
               "ms_per_step": ms_e2e / args.steps, "clocks": clocks_e2e}
    peak, peak_src = load_peaks()
    achieved = BYTES_PER_FAMILY * F / (trav_ms / 1e3) / 1e9
    traffic, traffic_src = ncu_traffic(f"cfg{args.config}")
    # FP64 side of the roofline: the walk's algorithmic Givens flops (Eq.13 over this rank's share
    # of the lattice) per walk time, against the measured FP64 FMA peak
    fl = eq13_flops(m) * F / total
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "traffic_source": traffic_src,
            "kernel": "walk_kernel (all shared-memory classes of a step)",
            "kernel_ms": trav_ms, "algorithmic_bytes_per_launch": BYTES_PER_FAMILY * F,
            "peak_source": peak_src,
            "store_peak": STORE_PEAK_GBS, "frac_of_store_peak": achieved / STORE_PEAK_GBS,
            "store_peak_source": "measured store-only bandwidth, coalesced 16 B stores (tools/microbench.cu, "
                                 "profiles/r01_microbench_b200.txt)",
            "fp64": {"algorithmic_flops_per_step": fl, "achieved_tflops": fl / (trav_ms / 1e3) / 1e12,
                     "peak_tflops": FP64_PEAK_TFLOPS, "frac": fl / (trav_ms / 1e3) / 1e12 / FP64_PEAK_TFLOPS,
                     "t_fp64_ms": fl / (FP64_PEAK_TFLOPS * 1e12) * 1e3,
                     "t_hbm_ms": BYTES_PER_FAMILY * F / (peak * 1e9) * 1e3,
                     "note": "Eq.13 Givens flops (PAPER.md:235-239, G6); peak = measured DFMA throughput "
                             "(tools/microbench.cu); the HBM term binds by ~14x"},
            "step_frac": (BYTES_PER_FAMILY * total * args.steps / (ms / 1e3) / 1e9) / peak / world}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, done, el, cores, o2 = oracle_rate(X, args.cpu_seconds)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
               "sample": f"{done} families uniformly sampled from cfg{args.config}'s {total} "
                         f"(O1 per-family Householder QR, n={n}), {el:.1f} s on the host",
               "full_table_s_extrapolated": total / rate,
               "reduced_oracle_O2": {"value": o2, "unit": UNIT,
                                     "sample": "1e6 of the same families, Householder on slices of the "
                                               "oracle's root QR (SURVEY.md §8(c) O2)"}}
    launches = args.steps * (h.launches_per_run() + (2 if rank == 0 else 0) + (1 if world > 1 else 0))
    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "f64",
               "data": "synthetic (seeded linear-Gaussian DAG, BASELINE.json configs recipe; datagen/)",
               "config": {"workload": f"cfg{args.config}", "m": m, "n": n,
                          "seed": args.seed if args.seed is not None else 1000 * args.config + 1,
                          "families": total, "k": plan["k"], "pinned": plan["b"], "tree_levels_global": plan["L1"],
                          "packs": plan["npacks"], "parallelism": f"lattice-sharded x{world}",
                          "pipeline": ("dataset s+1 loaded (H2D, centre, root QR, R broadcast, seed tree) on a "
                                       "second stream while dataset s is walked" if load_stream is not None
                                       else "none"),
                          "layout": ("(RSS, BIC) 16 B records, one table (bnreg_run_pairs)" if pairs else
                                     "separate RSS and BIC tables (bnreg_run)"),
                          "l2": "outputs (16 B/family, %.1f GB) >> L2 126 MB: every step evicts L2" % (
                              BYTES_PER_FAMILY * total / 1e9)},
               "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks, "gpu_launches": launches,
               "ms_per_step_recheck": ms_chk / args.steps, "run_ms_device": run_ms, "phases": phases}
        if sim:
            out["sim"] = {"world": args.sim_world, "rank": args.sim_rank, "rank_families": F,
                          "note": "one logical rank on one GPU, no collectives; value = this rank's families/s "
                                  "(every logical rank loads and factors X itself)"}
        print(json.dumps(out), flush=True)
    h.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        bench_reference(args)
    else:
        bench_ours(args)


if __name__ == "__main__":
    main()
