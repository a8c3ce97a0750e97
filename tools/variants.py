#!/usr/bin/env python
"""A/B variant builds of libbnreg.so: each variant = a set of -D defines, built to
tmpvar/lib_<name>.so (never over the in-tree library; load one with BNREG_LIB=...).

  python tools/variants.py build NAME=-DX,-DY NAME2= ...     (here, no GPU)
  python tools/variants.py run [--config C] [--reps R] NAME ... (on the GPU box: bench
        each variant's walk kernel time, alternating variants per repetition)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VAR = os.path.join(ROOT, "tmpvar")


def build(specs):
    from paper_1901_07643_b200 import build as b
    os.makedirs(VAR, exist_ok=True)
    for spec in specs:
        name, _, defs = spec.partition("=")
        defines = [d for d in defs.split(",") if d]
        out = os.path.join(VAR, f"lib_{name}.so")
        b.build(out=out, defines=defines)
        print(name, defines, "->", out, flush=True)


def run(args):
    cfg, reps, names = 5, 2, []
    it = iter(args)
    for a in it:
        if a == "--config":
            cfg = int(next(it))
        elif a == "--reps":
            reps = int(next(it))
        else:
            names.append(a)
    res = {n: [] for n in names}
    for r in range(reps):
        for n in names:
            env = dict(os.environ, BNREG_LIB=os.path.join(VAR, f"lib_{n}.so"))
            p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", str(cfg), "--steps", "5",
                                "--warmup", "3", "--no-e2e", "--no-cpu-baseline"], capture_output=True, text=True,
                               env=env, timeout=600)
            try:
                d = json.loads(p.stdout.strip().splitlines()[-1])
                res[n].append((d["ms_per_step"], d["roofline"]["kernel_ms"]))
                print(f"{n:14s} rep {r}: step {d['ms_per_step']:.3f} ms  walk {d['roofline']['kernel_ms']:.3f} ms"
                      f"  frac {d['roofline']['frac']:.3f}", flush=True)
            except Exception:
                print(n, "FAILED", p.stderr[-2000:], flush=True)
    for n in names:
        if res[n]:
            print(f"== {n:14s} best step {min(x[0] for x in res[n]):.3f}  best walk {min(x[1] for x in res[n]):.3f}")


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:])
    else:
        run(sys.argv[2:])
