"""Timeline of the pipelined step (DESIGN.md §4 "pipelined datasets"): CUDA events on the
run stream (walk) and the load stream (next dataset's prep), all relative to the first.
usage: python tools/overlap_probe.py [config] [steps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_1901_07643_b200 as bn  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
X = datagen.config_data(cfg, 5000 + cfg)
n, m = X.shape
dev = torch.device("cuda", 0)
h = bn.Bnreg(n, m, bn.options())
mode = os.environ.get("PROBE_STREAMS", "pool")
if mode == "prio":          # the load stream at high priority
    run_s, load_s = torch.cuda.Stream(dev), torch.cuda.Stream(dev, priority=-1)
elif mode == "raw":         # streams created by the runtime directly (not torch's pool)
    from cuda.bindings import runtime as rt
    raw = [rt.cudaStreamCreateWithFlags(rt.cudaStreamNonBlocking)[1] for _ in range(2)]
    run_s, load_s = (torch.cuda.ExternalStream(int(r), device=dev) for r in raw)
else:
    run_s, load_s = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
h.set_stream(run_s.cuda_stream)
h.set_load_stream(load_s.cuda_stream)
tab = torch.empty((h.num_families(), 2), dtype=torch.float64, device=dev)
bm = torch.empty(m, dtype=torch.int32, device=dev)
bb = torch.empty(m, dtype=torch.float64, device=dev)
Xd = torch.from_numpy(np.ascontiguousarray(X.T)).to(dev)
torch.cuda.synchronize()
ev = []


def mark(stream, name):
    e = torch.cuda.Event(enable_timing=True)
    e.record(stream)
    ev.append((name, e))


mark(run_s, "origin")
load_s.wait_stream(run_s)
import time
host = []
for s in range(steps):
    mark(load_s, f"prep{s}.begin")
    t = time.perf_counter()
    h.load_async(Xd)
    host.append((f"load{s}", time.perf_counter() - t))
    mark(load_s, f"prep{s}.end")
    mark(run_s, f"run{s}.begin")
    t = time.perf_counter()
    h.run_pairs_async(tab, bm.data_ptr(), bb.data_ptr())
    host.append((f"run{s}", time.perf_counter() - t))
    mark(run_s, f"run{s}.end")
torch.cuda.synchronize()
print("host ms per call:", " ".join(f"{k}={1e3 * v:.2f}" for k, v in host))
h.sync()
t0 = ev[0][1]
for name, e in ev[1:]:
    print(f"{name:14s} {t0.elapsed_time(e):9.3f} ms")
