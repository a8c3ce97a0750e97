import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import datagen, paper_1901_07643_b200 as bn
X = datagen.config_data(5); n, m = X.shape
for mode in ["direct", "levels"]:
    if mode == "levels": os.environ["BNREG_TREE_LEVELS"] = "1"
    h = bn.Bnreg.create(X); F = h.num_families()
    rss = torch.full((F,), float("nan"), dtype=torch.float64, device="cuda")
    bic = torch.full((F,), float("nan"), dtype=torch.float64, device="cuda")
    bm, bb = h.run(rss, bic); torch.cuda.synchronize(); h.close()
    nr = torch.isnan(rss).sum().item(); nb = torch.isnan(bic).sum().item()
    ninf = torch.isinf(bic).sum().item(); nneg = (rss <= 0).sum().item()
    print(mode, "nan rss", nr, "nan bic", nb, "inf bic", ninf, "rss<=0", nneg, flush=True)
    if nb:
        idx = torch.nonzero(torch.isnan(bic)).flatten()[:10].cpu().numpy()
        for i in idx:
            v = i >> (m - 1); c = i & ((1 << (m - 1)) - 1)
            print("  idx", i, "child", v, "cmask", hex(c), "rss", rss[i].item())
    del rss, bic; torch.cuda.empty_cache()
