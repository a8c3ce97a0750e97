"""Does a small kernel on another stream run beside the walk?  A 1-ms spin kernel
(tools/spin.cu, built on first use; CTAs x threads, smem bytes) launched on a second
stream right after the walk (bnreg_run_pairs_async): its end time relative to the walk's
start (DESIGN.md §4 "background prep").  The first launch of the spin kernel also pays
its lazy module load, which waits for the running walk."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_1901_07643_b200 as bn  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "spin.so")
if not os.path.exists(SO):
    import subprocess
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC", "-shared",
                           "-o", SO, os.path.join(HERE, "spin.cu")])
spin = ctypes.CDLL(SO)
X = datagen.config_data(5, 5005)
n, m = X.shape
dev = torch.device("cuda", 0)
h = bn.Bnreg(n, m, bn.options())
a, b = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
h.set_stream(a.cuda_stream)
tab = torch.empty((h.num_families(), 2), dtype=torch.float64, device=dev)
Xd = torch.from_numpy(np.ascontiguousarray(X.T)).to(dev)
h.load(Xd)
h.run_pairs_async(tab)
torch.cuda.synchronize()
for ctas, threads, smem in [(148, 32, 0), (148, 64, 0), (148, 64, 13000), (148, 64, 30000), (148, 128, 0)]:
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record(a)
    b.wait_event(e[0])
    h.run_pairs_async(tab)
    e[1].record(a)
    spin.spin_launch(ctypes.c_void_p(b.cuda_stream), ctypes.c_longlong(1000000), ctas, threads, smem)
    e[2].record(b)
    torch.cuda.synchronize()
    print(f"spin {ctas}x{threads} smem {smem}: walk end {e[0].elapsed_time(e[1]):.3f} ms, spin end {e[0].elapsed_time(e[2]):.3f} ms")
