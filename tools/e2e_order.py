"""Is the e2e/device gap an ordering (power/thermal) effect?  Alternate the two step kinds."""
import os, sys, time
import numpy as np, torch
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, R)
import datagen, paper_1901_07643_b200 as bn
X = datagen.config_data(5); n, m = X.shape
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
h = bn.Bnreg(n, m); h.set_stream(s.cuda_stream)
F = h.num_families(); tab = torch.empty((F, 2), dtype=torch.float64, device="cuda")
Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
Xpin = torch.from_numpy(np.ascontiguousarray(X.T)).pin_memory(); Xp = Xpin.numpy().T
bmd = torch.empty(m, dtype=torch.int32, device="cuda"); bbd = torch.empty(m, dtype=torch.float64, device="cuda")
def dev():
    h.load(Xd.data_ptr()); h.run_pairs_async(tab, bmd, bbd)
def e2e():
    h.load(Xp); h.run_pairs(tab)
def t(f, k=5):
    f(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(k): f()
    e1.record(s); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / k, 3)
h.timing(1)
for rep in range(3):
    print("device(timing)", t(dev), "e2e", t(e2e), "device(timing)", t(dev))
