import sys, numpy as np, torch
sys.path.insert(0, '.')
import datagen, paper_1901_07643_b200 as bn
X = datagen.config_data(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
h = bn.Bnreg.create(X)
F = h.num_families()
r = torch.empty(F, dtype=torch.float64, device='cuda'); b = torch.empty(F, dtype=torch.float64, device='cuda')
h.run(r, b); h.run(r, b)
