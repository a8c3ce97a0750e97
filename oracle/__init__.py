"""bnreg oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  It is independent of the CUDA path
(paper_1901_07643_b200/): neither imports the other, they share no code.

  oracle.c      -- O1/O2 per-family Householder regressions, BIC, argmax
                   (numerics; see its header for the passage each follows)
  schedule.py   -- the paper's combinatorics written out plainly: Alg.1
                   GreedySwaps, Eq.5 models of a permutation, Eq.9/Eq.13
                   counts, Alg.2 SeedPathCalculator

Parity status: every function here is pinned by a `-m "not gpu"` test in
tests/test_oracle_pins.py or tests/test_schedule_pins.py against something
other than itself (exact rational arithmetic, closed forms, the paper's printed
traces).  None is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc, -O2, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-D_GNU_SOURCE",
               "-o", tmp, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(tmp, _LIB)        # atomic: a process that has the old library mapped keeps it
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        i64, i32, u32, dbl = ctypes.c_int64, ctypes.c_int, ctypes.c_uint32, ctypes.c_double
        P = ctypes.c_void_p
        L.oracle_index.argtypes = [i32, i32, u32]
        L.oracle_index.restype = i64
        L.oracle_mask_of.argtypes = [i32, i64, ctypes.POINTER(ctypes.c_int)]
        L.oracle_mask_of.restype = u32
        L.oracle_centre.argtypes = [P, i64, i32, P]
        L.oracle_centre.restype = i32
        L.oracle_householder_rss.argtypes = [P, i64, i32]
        L.oracle_householder_rss.restype = dbl
        L.oracle_rss.argtypes = [P, i64, i32, i32, u32, P]
        L.oracle_rss.restype = dbl
        L.oracle_rss_residual.argtypes = [P, i64, i32, i32, u32]
        L.oracle_rss_residual.restype = dbl
        L.oracle_qr_r.argtypes = [P, i64, i32, P]
        L.oracle_qr_r.restype = None
        L.oracle_rss_reduced.argtypes = [P, i32, i32, u32]
        L.oracle_rss_reduced.restype = dbl
        L.oracle_bic.argtypes = [dbl, i64, i32]
        L.oracle_bic.restype = dbl
        L.oracle_score.argtypes = [dbl, i64, i32, i32]
        L.oracle_score.restype = dbl
        L.oracle_table.argtypes = [P, i64, i32, P, P, i32]
        L.oracle_table.restype = None
        L.oracle_rss_indices.argtypes = [P, i64, i32, P, i64, P, i32]
        L.oracle_rss_indices.restype = None
        L.oracle_rss_reduced_indices.argtypes = [P, i32, P, i64, P, i32]
        L.oracle_rss_reduced_indices.restype = None
        L.oracle_best.argtypes = [P, i32, P, P]
        L.oracle_best.restype = None
        L.oracle_reduced_table.argtypes = [P, i32, i64, P, P, i32]
        L.oracle_reduced_table.restype = None
        L.oracle_best_reduced.argtypes = [P, i32, i64, P, P, P, P, P, i32]
        L.oracle_best_reduced.restype = None
        L.oracle_num_threads.argtypes = []
        L.oracle_num_threads.restype = i32
        _lib = L
    return _lib


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def num_threads() -> int:
    return lib().oracle_num_threads()


def index(m: int, child: int, mask: int) -> int:
    return lib().oracle_index(m, child, mask)


def mask_of(m: int, idx: int):
    c = ctypes.c_int(0)
    s = lib().oracle_mask_of(m, idx, ctypes.byref(c))
    return c.value, s


def centre(X):
    """a1: column-major (n, m) -> centred copy (column-major)."""
    X = np.asfortranarray(X, dtype=np.float64)
    n, m = X.shape
    Xc = np.zeros((n, m), order="F")
    st = lib().oracle_centre(_ptr(X), n, m, _ptr(Xc))
    if st != 0:
        raise ValueError("non-finite input")
    return Xc


def rss(Xc, child: int, mask: int) -> float:
    Xc = np.asfortranarray(Xc, dtype=np.float64)
    n, m = Xc.shape
    return lib().oracle_rss(_ptr(Xc), n, m, child, mask, None)


def rss_residual(Xc, child: int, mask: int) -> float:
    Xc = np.asfortranarray(Xc, dtype=np.float64)
    n, m = Xc.shape
    return lib().oracle_rss_residual(_ptr(Xc), n, m, child, mask)


def qr_r(Xc):
    Xc = np.asfortranarray(Xc, dtype=np.float64)
    n, m = Xc.shape
    R = np.zeros((m, m))
    lib().oracle_qr_r(_ptr(Xc), n, m, _ptr(R))
    return R


def rss_reduced(R0, child: int, mask: int) -> float:
    R0 = _f64(R0)
    return lib().oracle_rss_reduced(_ptr(R0), R0.shape[0], child, mask)


def bic(rss_value: float, n: int, k: int) -> float:
    return lib().oracle_bic(float(rss_value), n, k)


SCORE_BIC, SCORE_AIC, SCORE_LL = 0, 1, 2


def _user_mask(c: int, v: int) -> int:
    lo = c & ((1 << v) - 1)
    return lo | ((c >> v) << (v + 1))


def _g14_better(s1, S1, s2, S2) -> bool:
    """G14: larger score, then smaller |S|, then smaller mask."""
    if s1 != s2:
        return s1 > s2
    p1, p2 = bin(S1).count("1"), bin(S2).count("1")
    return p1 < p2 if p1 != p2 else S1 < S2


def best_subsets_brute(scores, m: int):
    """SURVEY §8(f) NEXT 3, the plain definition (small m only): for every child v and
    candidate set C (table index of (v, C)), the best score over all S subset of C and
    that S (user ids), G14 tie-break.  Enumerates the subsets of every C."""
    scores = np.asarray(scores, dtype=np.float64)
    F = m << (m - 1)
    out_s = np.empty(F)
    out_m = np.empty(F, dtype=np.uint32)
    for v in range(m):
        for c in range(1 << (m - 1)):
            bs, bm = None, None
            sub = c
            while True:
                sc = scores[(v << (m - 1)) + sub]
                S = _user_mask(sub, v)
                if bs is None or _g14_better(sc, S, bs, bm):
                    bs, bm = sc, S
                if sub == 0:
                    break
                sub = (sub - 1) & c
            out_s[(v << (m - 1)) + c] = bs
            out_m[(v << (m - 1)) + c] = bm
    return out_s, out_m


def best_subsets(scores, m: int):
    """The same by the subset-max recursion bps(v, C) = best(score(v, C), bps(v, C - {u}))
    taken one bit at a time (Silander & Myllymaki's step), vectorised; pinned against
    best_subsets_brute.  Compressed masks keep the order and popcount of user masks, so
    G14 compares them directly."""
    scores = np.asarray(scores, dtype=np.float64)
    nb = m - 1
    out_s = scores.reshape(m, 1 << nb).copy()
    c = np.tile(np.arange(1 << nb, dtype=np.int64), (m, 1))
    pop = np.vectorize(lambda x: bin(int(x)).count("1"))
    popc = pop(np.arange(1 << nb)).astype(np.int64)
    for b in range(nb):
        idx = np.arange(1 << nb)
        hi = idx[(idx >> b) & 1 == 1]
        lo = hi ^ (1 << b)
        sj, si = out_s[:, lo], out_s[:, hi]
        cj, ci = c[:, lo], c[:, hi]
        pj, pi = popc[cj], popc[ci]
        better = (sj > si) | ((sj == si) & ((pj < pi) | ((pj == pi) & (cj < ci))))
        out_s[:, hi] = np.where(better, sj, si)
        c[:, hi] = np.where(better, cj, ci)
    v = np.arange(m)[:, None]
    lm = (np.int64(1) << v) - 1
    um = (c & lm) | ((c & ~lm) << 1)
    return out_s.reshape(-1), um.reshape(-1).astype(np.uint32)


def coefficients(Xc, child: int, mask: int):
    """Least-squares coefficients of child on the parent set `mask` ("solve
    the regression equations for each family"): the plain
    definition on the centred data, argmin_b ||x_v - X_S b||, by numpy's lstsq
    (a library primitive).  Returns a length-m vector (0 outside the set)."""
    Xc = np.asarray(Xc, dtype=np.float64)
    m = Xc.shape[1]
    S = [u for u in range(m) if (mask >> u) & 1 and u != child]
    beta = np.zeros(m)
    if S:
        b, *_ = np.linalg.lstsq(Xc[:, S], Xc[:, child], rcond=None)
        beta[S] = b
    return beta


def score(rss_value: float, n: int, k: int, kind: int) -> float:
    """oracle_score: BIC (0), AIC as loglik - k (1), log-likelihood (2); SURVEY §8(f) NEXT 4."""
    return lib().oracle_score(float(rss_value), n, k, kind)


def score_array(rss_arr, n: int, ks, kind: int):
    f = lib().oracle_score
    return np.array([f(float(r), n, int(k), kind) for r, k in zip(rss_arr, ks)])


def bic_array(rss_arr, n: int, ks):
    f = lib().oracle_bic
    return np.array([f(float(r), n, int(k)) for r, k in zip(rss_arr, ks)])


def table(Xc, want_bic: bool = True, threads: int = 0):
    """O1 over all m*2^(m-1) families -> (rss, bic) flat arrays."""
    Xc = np.asfortranarray(Xc, dtype=np.float64)
    n, m = Xc.shape
    total = m << (m - 1)
    r = np.zeros(total)
    b = np.zeros(total) if want_bic else None
    lib().oracle_table(_ptr(Xc), n, m, _ptr(r), _ptr(b) if want_bic else None, threads)
    return r, b


def rss_indices(Xc, idx, threads: int = 0):
    Xc = np.asfortranarray(Xc, dtype=np.float64)
    n, m = Xc.shape
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    out = np.zeros(len(idx))
    lib().oracle_rss_indices(_ptr(Xc), n, m, _ptr(idx), len(idx), _ptr(out), threads)
    return out


def rss_reduced_indices(R0, idx=None, threads: int = 0):
    R0 = _f64(R0)
    m = R0.shape[0]
    if idx is None:
        out = np.zeros(m << (m - 1))
        lib().oracle_rss_reduced_indices(_ptr(R0), m, None, 0, _ptr(out), threads)
    else:
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        out = np.zeros(len(idx))
        lib().oracle_rss_reduced_indices(_ptr(R0), m, _ptr(idx), len(idx), _ptr(out), threads)
    return out


def masks_of(m: int, idx):
    """Vectorised mask_of (same formula as oracle_mask_of, for numpy arrays)."""
    idx = np.asarray(idx, dtype=np.int64)
    v = idx >> (m - 1)
    c = idx & ((1 << (m - 1)) - 1)
    lo = c & ((np.int64(1) << v) - 1)
    hi = c >> v
    return v, (lo | (hi << (v + 1))).astype(np.int64)


def best(bic_table, m: int):
    """G14 argmax per child over a full table -> (masks uint32[m], bics f64[m])."""
    b = _f64(bic_table)
    bm = np.zeros(m, dtype=np.uint32)
    bb = np.zeros(m)
    lib().oracle_best(_ptr(b), m, _ptr(bm), _ptr(bb))
    return bm, bb


def best_reduced(R0, n: int, threads: int = 0):
    """oracle_best_reduced: per child, over all 2^(m-1) parent sets, the G14 best by O2 RSS
    and BIC, and the runner-up, without storing the table.  Returns a dict of arrays:
    best_mask, best_bic, best_rss, second_mask, second_bic."""
    R0 = _f64(R0)
    m = R0.shape[0]
    bm = np.zeros(m, dtype=np.uint32)
    bb = np.zeros(m)
    br = np.zeros(m)
    sm = np.zeros(m, dtype=np.uint32)
    sb = np.zeros(m)
    lib().oracle_best_reduced(_ptr(R0), m, n, _ptr(bm), _ptr(bb), _ptr(br), _ptr(sm), _ptr(sb), threads)
    return {"best_mask": bm, "best_bic": bb, "best_rss": br, "second_mask": sm, "second_bic": sb}


def reduced_table(R0, n: int, want_bic: bool = True, threads: int = 0):
    """O2 RSS and its BIC over all m*2^(m-1) families (oracle_reduced_table)."""
    R0 = _f64(R0)
    m = R0.shape[0]
    total = m << (m - 1)
    r = np.empty(total)
    b = np.empty(total) if want_bic else None
    lib().oracle_reduced_table(_ptr(R0), m, n, _ptr(r), _ptr(b) if want_bic else None, threads)
    return r, b
