import os, sys, time
import numpy as np, torch
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, R)
import datagen, paper_1901_07643_b200 as bn
X = datagen.config_data(5); n, m = X.shape
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
h = bn.Bnreg(n, m); h.set_stream(s.cuda_stream)
F = h.num_families(); tab = torch.empty((F, 2), dtype=torch.float64, device="cuda")
Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
bmd = torch.empty(m, dtype=torch.int32, device="cuda"); bbd = torch.empty(m, dtype=torch.float64, device="cuda")
h.load(Xd.data_ptr()); torch.cuda.synchronize()
small = torch.zeros(1024, device="cuda")
def t(f, k=5):
    f(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter(); e0.record(s)
    for _ in range(k): f()
    e1.record(s); torch.cuda.synchronize(); w1 = time.perf_counter()
    return round(e0.elapsed_time(e1) / k, 3), round((w1 - w0) * 1e3 / k, 3)
print("tiny kernel + sync", t(lambda: (small.add_(1), s.synchronize()), 50))
print("async back-to-back", t(lambda: h.run_pairs_async(tab, bmd, bbd)))
print("async + stream sync", t(lambda: (h.run_pairs_async(tab, bmd, bbd), s.synchronize())))
def with_evt():
    e = torch.cuda.Event(enable_timing=True); h.run_pairs_async(tab, bmd, bbd); e.record(s); e.synchronize()
print("async + event sync", t(with_evt))
# where does the time go: per-iteration events around the run
es = []
for _ in range(5):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(s); h.run_pairs_async(tab, bmd, bbd); b.record(s); b.synchronize(); es.append(a.elapsed_time(b))
print("bracketed single run (ms)", [round(x, 3) for x in es])
h.timing(1)
es = []
for _ in range(5):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(s); h.run_pairs_async(tab, bmd, bbd); b.record(s); b.synchronize(); es.append(a.elapsed_time(b))
tms, runs = h.timing(0)
print("bracketed single run, handle timing on (ms)", [round(x, 3) for x in es], "handle whole", round(tms[0] / runs, 3))
es = []
for _ in range(5):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(s); h.run_pairs(tab); b.record(s); b.synchronize(); es.append(a.elapsed_time(b))
print("bracketed run_pairs (sync)", [round(x, 3) for x in es])
es = []
for _ in range(5):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(s); h.run_pairs_async(tab, bmd, bbd); h.run_pairs_async(tab, bmd, bbd); b.record(s); b.synchronize(); es.append(a.elapsed_time(b) / 2)
print("bracketed 2 runs (per run)", [round(x, 3) for x in es])
