"""CPU-side checks of the C-ABI library: it loads, exports every symbol
include/bnreg.h declares, and its host logic (schedule, indexing, plan,
partition, best merge) agrees with the paper / oracle combinatorics.
No compute call here needs a GPU."""
import itertools
import os
import re

import numpy as np
import pytest

import oracle
from oracle import schedule as sc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bn():
    import paper_1901_07643_b200 as bn
    from paper_1901_07643_b200 import build
    build.build()
    bn.lib()
    return bn


def test_exports_every_declared_symbol(bn):
    hdr = open(os.path.join(ROOT, "include", "bnreg.h")).read()
    declared = set(re.findall(r"\b(bnreg_[a-z_]+)\s*\(", hdr))
    assert declared == set(bn.SYMBOLS), declared ^ set(bn.SYMBOLS)
    L = bn.lib()
    for s in declared:
        assert getattr(L, s) is not None


def test_schedule_matches_paper(bn):
    for k in range(2, 17):
        assert bn.bnreg_schedule(k).tolist() == sc.greedy_swaps(k)
    with pytest.raises(ValueError):
        bn.bnreg_schedule(1)


def test_index_matches_oracle(bn):
    rng = np.random.default_rng(0)
    for _ in range(2000):
        m = int(rng.integers(2, 31))
        v = int(rng.integers(0, m))
        S = int(rng.integers(0, 1 << m))
        assert bn.bnreg_index(m, v, S) == oracle.index(m, v, S)


@pytest.mark.parametrize("m,k", [(8, 4), (12, 5), (16, 8), (20, 8), (28, 8), (24, 7)])
def test_plan_partition(bn, m, k):
    """Packs x 2^p workers enumerate every Alg.2 worker (every front set of the
    pinned variables) exactly once; world ranks split packs disjointly with
    equal cost (complementary top-bit patterns)."""
    n = 1000
    q = bn.bnreg_plan_query(m, n, bn.options(free_vars=k))
    assert q["sched_len"] == 2 ** k - k - 1
    assert q["b"] == m - k and q["p"] == min(3, m - k)   # 8 lockstep workers per warp (walk kernel)
    def expand(items):
        gs = q["bh"] - q["g"]
        return [it | (j << gs) for it in items for j in range(1 << q["g"])]

    packs = expand(bn.bnreg_plan_packs(m, n, bn.options(free_vars=k)).tolist())
    assert sorted(packs) == list(range(1 << q["bh"]))
    for world in [2, 4, 8]:
        if (1 << (q["bh"] - q["g"])) < 2 * world:
            continue
        allp, costs, fams = [], [], 0
        for rank in range(world):
            o = bn.options(free_vars=k, world=world, rank=rank)
            pr = expand(bn.bnreg_plan_packs(m, n, o).tolist())
            allp += pr
            # family count of a pack = sum over its workers of 2^(k-1)(2(m-d)-k) (V11)
            c = sum(sum(2 ** (k - 1) * (2 * (m - (bin(P).count("1") + bin(w).count("1"))) - k)
                        for w in range(1 << q["p"])) for P in pr)
            costs.append(c)
            fams += bn.bnreg_plan_query(m, n, o)["local_families"]
        assert sorted(allp) == list(range(1 << q["bh"]))
        assert len(set(costs)) == 1 and costs[0] * world == m << (m - 1)
        assert fams == m << (m - 1)


def test_worker_family_counts_match_alg2(bn):
    """The B200 relabelling is Alg.2 with pinned set {0,1} u {hi ids}: the
    per-worker family counts of the plan equal those of seed_path workers."""
    m, k = 9, 4
    b = m - k
    counts_paper = sorted(len(sc.worker_owned_families(list(bits), m))
                          for bits in itertools.product([0, 1], repeat=b))
    q = bn.bnreg_plan_query(m, 100, bn.options(free_vars=k))
    counts_plan = sorted(2 ** (k - 1) * (2 * (m - (bin(P).count("1") + bin(w).count("1"))) - k)
                         for P in range(1 << q["bh"]) for w in range(1 << q["p"]))
    assert counts_paper == counts_plan


def test_plan_errors(bn):
    with pytest.raises(bn.BnregError):
        bn.bnreg_plan_query(1, 100)
    with pytest.raises(bn.BnregError):
        bn.bnreg_plan_query(8, 5)             # n < m + 1
    with pytest.raises(bn.BnregError):
        bn.bnreg_plan_query(8, 100, bn.options(free_vars=1))
    with pytest.raises(bn.BnregError):
        bn.bnreg_plan_query(8, 100, bn.options(world=3))
    with pytest.raises(bn.BnregError):
        bn.bnreg_plan_query(6, 100, bn.options(free_vars=5, world=8))


def test_best_merge(bn):
    m = 3
    masks = np.array([[2, 0xFFFFFFFF, 1], [4, 5, 3]], dtype=np.uint32)
    bics = np.array([[-1.0, 0.0, -2.0], [-1.0, -3.0, -2.0]])
    om, ob = bn.bnreg_best_merge(m, masks, bics)
    assert om.tolist() == [2, 5, 1]           # tie on BIC and |S| -> smaller mask; tie on BIC -> smaller |S|
    assert ob.tolist() == [-1.0, -3.0, -2.0]


def test_walk_rejects_large_k(bn):
    """The walk kernel takes k <= 8 free variables (a step's free list is one u32 of
    nibbles, at most 2 entries per lane)."""
    with pytest.raises(bn.BnregError):
        bn.bnreg_plan_query(24, 1000, bn.options(free_vars=9))


def test_null_handle_is_rejected(bn):
    """include/bnreg.h: every call taking a handle returns BNREG_E_INVAL (1) for a NULL
    handle, with a message in bnreg_last_error, before touching the device (no GPU
    needed); the int64 queries return -1 and bnreg_destroy(NULL) is a no-op."""
    import ctypes
    L = bn.lib()
    checked = 0
    for name in bn.SYMBOLS:
        f = getattr(L, name)
        args = f.argtypes or []
        if not args or args[0] is not ctypes.c_void_p or name == "bnreg_create":
            continue
        vals = [None] + [0 if a in (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32) else None for a in args[1:]]
        r = f(*vals)
        if f.restype is ctypes.c_int32:
            assert r == 1, name
            assert L.bnreg_last_error(), name
            checked += 1
        elif f.restype is ctypes.c_int64:
            assert r == -1, name
    assert checked >= 15
    L.bnreg_destroy(None)
