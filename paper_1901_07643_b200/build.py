"""Build libbnreg.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

The library is rebuilt whenever the sources, headers, nvcc flags or extra -D
defines differ from the ones recorded in libbnreg.stamp (a hash), so a copied-in
or variant build can never be mistaken for the committed sources.  Variant builds
(e.g. the K8 write-counting debug build) go to their own path (`out=`)."""
from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SOURCES = ["bnreg_api.cu", "bnreg_kernels.cu", "walk_pairs.cu", "walk_tables.cu", "walks_pairs.cu", "walks_tables.cu", "walk7_kernel.cu", "walk7_tables.cu", "seed_kernel.cu", "bps_kernel.cu"]
HEADERS = ["plan.h", "kernels.h", "device.cuh", "walk_kernel.cuh", "walks_kernel.cuh", "tmem.cuh"]
OUT = os.path.join(HERE, "libbnreg.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


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
    objdir = tempfile.mkdtemp(prefix="bnreg_obj_")
    try:
        # one nvcc per translation unit, in parallel (the walk kernel's instantiations
        # dominate: the record layout and the table layouts are separate units), then link
        procs, objs = [], []
        for src in SOURCES:
            o = os.path.join(objdir, src.replace(".cu", ".o"))
            objs.append(o)
            procs.append(subprocess.Popen([NVCC, *FLAGS, *defines, "-c", "-o", o, os.path.join(CSRC, src)],
                                          stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
        logs, bad = [], False
        for src, pr in zip(SOURCES, procs):
            so, se = pr.communicate()
            logs.append(f"== {src}\n{so}{se}")
            bad |= pr.returncode != 0
        if bad:
            sys.stderr.write("\n".join(logs))
            raise RuntimeError("nvcc failed")
        r = subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs, "-ldl"],
                           capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc link failed")
    finally:
        shutil.rmtree(objdir, ignore_errors=True)
    os.replace(tmp, out)             # atomic: a process that has the old library mapped keeps it
    if out == OUT:
        with open(os.path.join(HERE, "ptxas.log"), "w") as f:
            f.write("\n".join(logs))
    with open(st, "w") as f:
        f.write(dg + "\n")
    if verbose:
        sys.stderr.write("\n".join(logs))
    return out


K8_OUT = os.path.join(HERE, "libbnreg_k8.so")


def build_k8(force: bool = False) -> str:
    """The K8 debug build (per-entry write counters, bnreg_debug_write_counts)."""
    return build(force=force, out=K8_OUT, defines=["-DBNREG_K8=1"])


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
