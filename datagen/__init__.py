"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module holds NONE of the method's arithmetic (no QR, no Givens, no RSS):
it only draws the data matrices that BASELINE.json's configs describe, so that
the oracle (oracle/) and the CUDA path (paper_1901_07643_b200/) can be fed the
same bytes without sharing any code with each other.

Recipe (SURVEY.md §8(d) "Generator", BASELINE.json "configs"):
  1. order = rng.permutation(m)                       -- random topological order
  2. for a < b in topological order: an edge order[a] -> order[b] exists with
     probability p; its weight is sign * U(lo, hi) with sign = +-1 w.p. 1/2
     (reading G24)
  3. sigma_v = 1, or sigma_v ~ U(0.5, 2) per variable for cfg4 (reading G25)
  4. for v in topological order: X[:, v] = X @ W[:, v] + sigma_v * N(0, 1)^n
  5. cfg3 only: (i, j) = rng.choice(m, 2, replace=False);
     X[:, j] = X[:, i] + 1e-6 * N(0, 1)^n          -- near-collinear pair (G23)
The generator does NOT centre: centring is step a1 of the method and both the
oracle and the library do it themselves (BASELINE.json says the columns are
centred -- that is the method's job here).

Output: float64 array of shape (n, m) in column-major (Fortran) order, which is
the layout the C-ABI `bnreg_create` takes (ld = n).
"""
from __future__ import annotations

import numpy as np

# cfg id -> (m, n, edge prob, |w| low, |w| high, heteroscedastic, collinear pair)
CONFIGS = {
    1: dict(m=8, n=100, p=0.3, lo=0.5, hi=2.0, hetero=False, pair=False),
    2: dict(m=16, n=1000, p=0.2, lo=0.5, hi=2.0, hetero=False, pair=False),
    3: dict(m=20, n=5000, p=0.15, lo=0.5, hi=2.0, hetero=False, pair=True),
    4: dict(m=24, n=10000, p=0.1, lo=0.1, hi=3.0, hetero=True, pair=False),
    5: dict(m=28, n=2000, p=0.08, lo=0.5, hi=2.0, hetero=False, pair=False),
}


def dag_data(m: int, n: int, p: float, lo: float, hi: float, seed: int,
             hetero: bool = False, pair: bool = False, meta: dict | None = None):
    """Linear-Gaussian DAG sample, column-major (n, m) float64. See module doc."""
    if m < 1 or n < 1:
        raise ValueError("m, n must be positive")
    rng = np.random.default_rng(seed)
    order = rng.permutation(m)
    W = np.zeros((m, m))
    for a in range(m):
        for b in range(a + 1, m):
            if rng.random() < p:
                sign = 1.0 if rng.random() < 0.5 else -1.0
                W[order[a], order[b]] = sign * rng.uniform(lo, hi)
    sigma = rng.uniform(0.5, 2.0, m) if hetero else np.ones(m)
    X = np.zeros((n, m), order="F")
    for v in order:
        X[:, v] = X @ W[:, v] + sigma[v] * rng.standard_normal(n)
    pr = None
    if pair and m >= 2:
        i, j = (int(t) for t in rng.choice(m, 2, replace=False))
        X[:, j] = X[:, i] + 1e-6 * rng.standard_normal(n)
        pr = (i, j)
    if meta is not None:
        meta.update(order=order.tolist(), W=W, sigma=sigma, pair=pr, seed=seed)
    return np.asfortranarray(X)


def config_data(cfg: int, seed: int | None = None, meta: dict | None = None):
    """Data for BASELINE.json configs[cfg-1]; default seed 1000*cfg + 1 (§8(d))."""
    c = CONFIGS[cfg]
    if seed is None:
        seed = 1000 * cfg + 1
    return dag_data(c["m"], c["n"], c["p"], c["lo"], c["hi"], seed,
                    hetero=c["hetero"], pair=c["pair"], meta=meta)


def gaussian(n: int, m: int, seed: int, offset: float = 0.0):
    """i.i.d. N(0,1) + optional per-column offsets (exercises centring)."""
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, m))
    if offset:
        X = X + offset * rng.uniform(-1.0, 1.0, m)[None, :]
    return np.asfortranarray(X)


def sample_indices(m: int, count: int, seed: int):
    """Seeded uniform sample of flat table indices in [0, m*2^(m-1))."""
    rng = np.random.default_rng(seed)
    total = m * (1 << (m - 1))
    return np.sort(rng.choice(total, size=min(count, total), replace=False)).astype(np.int64)
