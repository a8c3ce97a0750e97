import sys, numpy as np
import os; R = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, 'tests'))
import datagen, oracle
import paper_1901_07643_b200 as bn
from gpu_util import run_tables
for k in [3, 2, 4]:
    X = datagen.config_data(1)
    Xc = oracle.centre(X); n, m = X.shape
    rss, bic, bm, bb, h = run_tables(X, bn.options(free_vars=k))
    ref, _ = oracle.table(Xc, want_bic=False)
    err = np.abs(rss - ref) / ref
    bad = np.nonzero(err > 1e-9)[0]
    print("k", k, "bad", len(bad))
    for i in bad[:20]:
        v, S = oracle.masks_of(m, np.array([i]))
        # find which reference entry equals the GPU value
        match = np.nonzero(np.abs(ref - rss[i]) / ref < 1e-9)[0]
        print(i, int(v[0]), format(int(S[0]), '08b'), rss[i], ref[i], "gpu value equals ref at", [(int(oracle.masks_of(m, np.array([j]))[0][0]), format(int(oracle.masks_of(m, np.array([j]))[1][0]), '08b')) for j in match[:3]])
    print(bn.bnreg_plan_query(m, n, bn.options(free_vars=k)))
    h.close()
