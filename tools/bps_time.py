"""Time bnreg_best_subsets at cfg5 (m=28) on the record table's BIC column."""
import os, sys
import numpy as np, torch
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, R)
import datagen, paper_1901_07643_b200 as bn
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
X = datagen.config_data(cfg); n, m = X.shape
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
h = bn.Bnreg.create(X); h.set_stream(s.cuda_stream)
F = h.num_families()
t = torch.empty((F, 2), dtype=torch.float64, device="cuda")
bs = torch.empty(F, dtype=torch.float64, device="cuda"); bm = torch.empty(F, dtype=torch.int32, device="cuda")
h.run_pairs(t)
for _ in range(2):
    h.best_subsets(t.data_ptr() + 8, 2, bs, bm)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(3):
    h.best_subsets(t.data_ptr() + 8, 2, bs, bm)
e1.record(s); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
nb = m - 1
R = max(0, nb - 12)
passes = 1 + (0 if R == 0 else (1 if R < 4 else (R + 7) // 8))
byts = F * 16 + F * 12 + (passes - 1) * F * 24      # low: read records, write (score, mask); groups: r+w
print(f"cfg{cfg} m={m}: best_subsets {ms:.2f} ms, {passes} passes, {byts / 1e9:.0f} GB moved, {byts / ms / 1e6:.0f} GB/s")
