"""Per-phase device time of a run: back-to-back vs after an idle GPU (cfg5, pairs)."""
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
for mode in ["idle-gap", "idle 50ms", "back-to-back"]:
    h.timing(1)
    for _ in range(5):
        h.run_pairs_async(tab, bmd, bbd)
        if mode == "idle-gap":
            torch.cuda.synchronize()
        if mode == "idle 50ms":
            torch.cuda.synchronize(); time.sleep(0.05)
    torch.cuda.synchronize()
    tms, runs = h.timing(0)
    print(mode, "runs", runs, "whole %.3f seeds %.3f walk %.3f reduce %.3f" % tuple(x / runs for x in tms))
