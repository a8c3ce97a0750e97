"""Where does the e2e step spend its time? (cfg5, pairs layout; handle on a torch side stream)"""
import os, sys, time
import numpy as np, torch
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, R)
import datagen, paper_1901_07643_b200 as bn
X = datagen.config_data(5); n, m = X.shape
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
h = bn.Bnreg(n, m); h.set_stream(s.cuda_stream)
F = h.num_families(); tab = torch.empty((F, 2), dtype=torch.float64, device="cuda")
Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
Xpin = torch.from_numpy(np.ascontiguousarray(X.T)).pin_memory(); Xp = Xpin.numpy().T
bmd = torch.empty(m, dtype=torch.int32, device="cuda"); bbd = torch.empty(m, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
def t(f, k=5):
    f(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter(); e0.record(s)
    for _ in range(k): f()
    e1.record(s); torch.cuda.synchronize(); w1 = time.perf_counter()
    return round(e0.elapsed_time(e1) / k, 3), round((w1 - w0) * 1e3 / k, 3)
print("stream", s.cuda_stream)
print("load(Xd)", t(lambda: h.load(Xd.data_ptr())))
print("load(Xpin)", t(lambda: h.load(Xp)))
print("run_pairs_async", t(lambda: h.run_pairs_async(tab, bmd, bbd)))
print("run_pairs best=False", t(lambda: h.run_pairs(tab, best=False)))
print("run_pairs (sync + D2H)", t(lambda: h.run_pairs(tab)))
print("device step", t(lambda: (h.load(Xd.data_ptr()), h.run_pairs_async(tab, bmd, bbd))))
print("e2e step", t(lambda: (h.load(Xp), h.run_pairs(tab))))
# host-side cost of issuing one run (GPU idle before)
ts = []
for _ in range(5):
    torch.cuda.synchronize()
    w0 = time.perf_counter(); h.run_pairs_async(tab, bmd, bbd); w1 = time.perf_counter()
    ts.append((w1 - w0) * 1e3)
torch.cuda.synchronize()
print("host issue time of run_pairs_async (ms)", [round(x, 3) for x in ts])
ts = []
for _ in range(5):
    torch.cuda.synchronize()
    w0 = time.perf_counter(); h.load(Xd.data_ptr()); w1 = time.perf_counter()
    ts.append((w1 - w0) * 1e3)
print("host time of load (ms)", [round(x, 3) for x in ts])
