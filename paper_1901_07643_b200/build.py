"""Build libbnreg.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

The library is rebuilt whenever the sources, headers, nvcc flags or extra -D
defines differ from the ones recorded in libbnreg.stamp (a hash), so a copied-in
or variant build can never be mistaken for the committed sources.  Variant builds
(e.g. the K8 write-counting debug build) go to their own path (`out=`)."""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SOURCES = ["bnreg_api.cu", "bnreg_kernels.cu", "walk_kernel.cu", "seed_kernel.cu", "bps_kernel.cu"]
HEADERS = ["plan.h", "kernels.h", "device.cuh"]
OUT = os.path.join(HERE, "libbnreg.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def _digest(defines) -> str:
    h = hashlib.sha256()
    for f in SOURCES + HEADERS:
        with open(os.path.join(CSRC, f), "rb") as fh:
            h.update(f.encode() + b"\0" + fh.read())
    with open(os.path.join(HERE, "..", "include", "bnreg.h"), "rb") as fh:
        h.update(fh.read())
    h.update(" ".join([NVCC, *FLAGS, *defines]).encode())
    return h.hexdigest()


def _stamp(out):
    return os.path.splitext(out)[0] + ".stamp"


def build(force: bool = False, verbose: bool = False, out: str = OUT, defines=()) -> str:
    defines = list(defines)
    dg = _digest(defines)
    st = _stamp(out)
    if not force and os.path.exists(out) and os.path.exists(st) and open(st).read().strip() == dg:
        return out
    tmp = out + f".tmp{os.getpid()}"
    cmd = [NVCC, *FLAGS, *defines, "-o", tmp, *[os.path.join(CSRC, s) for s in SOURCES]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed")
    os.replace(tmp, out)             # atomic: a process that has the old library mapped keeps it
    if out == OUT:
        with open(os.path.join(HERE, "ptxas.log"), "w") as f:
            f.write(r.stderr)
    with open(st, "w") as f:
        f.write(dg + "\n")
    if verbose:
        sys.stderr.write(r.stderr)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
