#!/usr/bin/env python
"""Write tests/golden/best_cfg{3,4,5}.json: the per-child argmax of the BIC over ALL
m*2^(m-1) families of BASELINE.json configs[2..4] (seeded datagen inputs), computed by
the oracle only (oracle.best_reduced: O2 per-family Householder on slices of the
oracle's own root QR + oracle_bic + the G14 tie-break, streamed; SURVEY.md §8(c)
"O2 full argmax at cfg4-5").  No value comes from the CUDA path.

Each record: child, best_mask, best_bic, best_rss, second_mask, second_bic and
gap = best_bic - second_bic (the G14 exemption rule needs the top-2 gap).

  OMP_NUM_THREADS=8 python tests/golden/make_best_golden.py [cfg ...]
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
import oracle  # noqa: E402


def main(cfgs):
    for cfg in cfgs:
        X = datagen.config_data(cfg)
        n, m = X.shape
        Xc = oracle.centre(X)
        R0 = oracle.qr_r(Xc)
        t0 = time.time()
        d = oracle.best_reduced(R0, n)
        el = time.time() - t0
        rows = []
        for v in range(m):
            rows.append({"child": v, "best_mask": int(d["best_mask"][v]), "best_bic": float(d["best_bic"][v]),
                         "best_rss": float(d["best_rss"][v]), "second_mask": int(d["second_mask"][v]),
                         "second_bic": float(d["second_bic"][v]),
                         "gap": float(d["best_bic"][v] - d["second_bic"][v])})
        out = {"config": cfg, "m": m, "n": n, "seed": 1000 * cfg + 1,
               "source": "oracle.best_reduced (O2 full table, oracle_bic, G14), tests/golden/make_best_golden.py",
               "families": m << (m - 1), "seconds": round(el, 1), "threads": oracle.num_threads(),
               "children": rows}
        with open(os.path.join(HERE, f"best_cfg{cfg}.json"), "w") as f:
            json.dump(out, f, indent=1)
        print(f"cfg{cfg}: {el:.1f} s, min gap {min(r['gap'] for r in rows):.3e}", flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [3, 4, 5])
