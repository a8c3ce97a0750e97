"""Root factor by TSQR vs Gram + Cholesky: load time and RSS accuracy on
the families of cfg3 that contain its near-collinear pair."""
import os, sys, time
import numpy as np, torch
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, R)
sys.path.insert(0, os.path.join(R, "tests"))
import datagen, oracle, paper_1901_07643_b200 as bn
for cfg in (3, 5):
    meta = {}
    X = datagen.config_data(cfg, meta=meta)
    n, m = X.shape
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
    for method, name in ((bn.ROOT_TSQR, "tsqr"), (bn.ROOT_CHOLESKY, "cholesky")):
        h = bn.Bnreg(n, m); h.set_root_method(method)
        for _ in range(3): h.load(Xd.data_ptr())
        torch.cuda.synchronize(); w0 = time.perf_counter()
        for _ in range(20): h.load(Xd.data_ptr())
        ms = (time.perf_counter() - w0) * 1e3 / 20
        line = f"cfg{cfg} {name}: load (centre + factor, synchronous) {ms:.3f} ms"
        if cfg == 3:
            i, j = meta["pair"]
            rng = np.random.default_rng(9)
            idx = sorted(set(oracle.index(m, v, (int(rng.integers(0, 1 << m)) | (1 << i) | (1 << j)) & ~(1 << v))
                             for v in rng.integers(0, m, 400) if v not in (i, j)))
            idx = np.array(idx, dtype=np.int64)
            ref = oracle.rss_indices(oracle.centre(X), idx)
            t = torch.empty((h.num_families(), 2), dtype=torch.float64, device="cuda")
            h.run_pairs(t); torch.cuda.synchronize()
            got = t[torch.from_numpy(idx).cuda(), 0].cpu().numpy()
            line += f", max rel RSS err on {len(idx)} pair families {np.abs(got - ref).max() / 1 if False else (np.abs(got - ref) / ref).max():.2e}"
        print(line)
        h.close()
