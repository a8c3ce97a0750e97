"""Host-side cost of one step's calls (load, run_pairs_async) vs the device time."""
import os, sys, time
import numpy as np, torch
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, R)
import datagen, paper_1901_07643_b200 as bn
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
X = datagen.config_data(cfg); n, m = X.shape
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
h = bn.Bnreg.create(X); h.set_stream(s.cuda_stream)
F = h.num_families()
tab = torch.empty((F, 2), dtype=torch.float64, device="cuda")
bm = torch.empty(m, dtype=torch.int32, device="cuda"); bb = torch.empty(m, dtype=torch.float64, device="cuda")
Xd = torch.from_numpy(np.asfortranarray(X)).cuda()
for _ in range(3):
    h.load(Xd); h.run_pairs_async(tab, bm, bb)
torch.cuda.synchronize()
tl, tr = [], []
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(10):
    t0 = time.perf_counter(); h.load(Xd); t1 = time.perf_counter(); h.run_pairs_async(tab, bm, bb); t2 = time.perf_counter()
    tl.append(t1 - t0); tr.append(t2 - t1)
e1.record(s); torch.cuda.synchronize()
print(f"cfg{cfg}: step {e0.elapsed_time(e1) / 10:.3f} ms; host load {np.median(tl) * 1e3:.3f} ms, run_pairs_async call {np.median(tr) * 1e3:.3f} ms")
e0.record(s)
for _ in range(10):
    h.run_pairs_async(tab, bm, bb)
e1.record(s); torch.cuda.synchronize()
print(f"cfg{cfg}: run only {e0.elapsed_time(e1) / 10:.3f} ms")
