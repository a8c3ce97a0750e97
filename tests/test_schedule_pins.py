"""Pins of the paper's combinatorics (oracle/schedule.py) against what the paper
prints and what exhaustive enumeration fixes."""
import itertools
import os

import pytest

from oracle import schedule as sc


def test_base_cases_alg1_eq7():
    assert sc.greedy_swaps(2) == [1]
    # Eq.7: GRC_1, GRC_2, GRC_1, GRC_2 walks ABC -> CAB
    assert sc.greedy_swaps(3) == [1, 2, 1, 2]
    perms = sc.walk(3, sc.greedy_swaps(3), start=list("ABC"))
    assert ["".join(p) for p in perms] == ["ABC", "BAC", "BCA", "CBA", "CAB"]
    # "all 9 regression models are included in this permutation set"
    assert sc.verify_coverage(3, sc.greedy_swaps(3)) == 9


def test_eq8_trace(golden_dir):
    rows = [l.split() for l in open(os.path.join(golden_dir, "eq8_trace.txt"))
            if l.strip() and not l.startswith("#")]
    printed_perms = [r[:4] for r in rows]
    printed_counts = [int(r[4]) for r in rows]
    perms = sc.walk(4, sc.greedy_swaps(4), start=list("ABCD"))
    assert perms == printed_perms
    counts = sc.cumulative_model_counts(4, sc.greedy_swaps(4))
    # exact enumeration differs from the print only at [D,B,A,C]: 27, not 26 (G22)
    diff = [i for i, (a, b) in enumerate(zip(counts, printed_counts)) if a != b]
    assert diff == [10] and counts[10] == 27 and printed_counts[10] == 26
    assert counts[-1] == 28 == sc.total_models(4)


def test_each_swap_adds_exactly_one_new_prefix_set():
    """every swap of Upsilon(m) exposes one never-seen prefix set;
    greedy productivity (>= 1 new model per swap)."""
    for m in range(2, 10):
        order = list(range(1, m + 1))
        seen_pref = {frozenset(order[:k]) for k in range(1, m)}
        seen = sc.models_of_permutation(order)
        for i in sc.greedy_swaps(m):
            order = sc.apply_swap(order, i)
            new = sc.new_models_after_swap(order, i, seen)
            assert len(new) == m - i >= 1
            pre = frozenset(order[:i])
            assert pre not in seen_pref
            seen_pref.add(pre)
            seen |= sc.models_of_permutation(order)
        assert len(seen_pref) == 2 ** m - 2


@pytest.mark.parametrize("m", range(2, 21))
def test_length_eq9(m):
    assert len(sc.greedy_swaps(m)) == sc.schedule_length(m) == 2 ** m - m - 1


@pytest.mark.parametrize("m", range(2, 11))
def test_coverage_complete(m):
    assert sc.verify_coverage(m, sc.greedy_swaps(m)) == sc.total_models(m)


def test_alg1_as_printed_fails_coverage():
    """Reading G2 / SURVEY V5: without the +1 the printed Alg.1 misses models."""
    assert sc.verify_coverage(3, sc.greedy_swaps_as_printed(3)) == 8
    assert sc.verify_coverage(4, sc.greedy_swaps_as_printed(4)) == 20
    assert sc.verify_coverage(6, sc.greedy_swaps_as_printed(6)) < sc.total_models(6)


def test_flops_eq13():
    """Eq.13 (read with G6) = sum of 6(m-i+1) over Upsilon(m) = Eq.11 recurrence."""
    assert sc.predicted_rotation_flops(2) == 12
    assert sc.predicted_rotation_flops(3) == 60
    assert sc.predicted_rotation_flops(10) == 36468   # SPEC.md:248 says 36474 (slip)
    for m in range(2, 17):
        f = sc.rotation_flops(m, sc.greedy_swaps(m))
        assert f == sc.predicted_rotation_flops(m) == sc.runtime_recurrence(m)
    assert sc.predicted_rotation_flops(28) == 24159188430


def test_minimality_exhaustive_m3_and_sampled_m4():
    """§4: 2^m - m - 1 swaps are the minimum."""
    for seq in itertools.product([1, 2], repeat=3):
        assert sc.verify_coverage(3, list(seq)) < 9
    import random
    rnd = random.Random(1)
    for _ in range(1500):
        seq = [rnd.randint(1, 3) for _ in range(10)]
        assert sc.verify_coverage(4, seq) < 28


def test_index_occurrences_binomial():
    """index i appears C(m,i) - 1 times in Upsilon(m)."""
    from math import comb
    for m in range(3, 13):
        s = sc.greedy_swaps(m)
        for i in range(1, m):
            assert s.count(i) == comb(m, i) - 1


def test_alg2_paper_p2_example_and_spec_examples():
    """core 0 = identity order with Upsilon0(m-1); core 1 =
    [v_m, v_1..v_{m-1}] with [i+1 | i in Upsilon0(m-1)]."""
    for m in range(3, 9):
        o0, d0, s0 = sc.seed_path([0], m)
        o1, d1, s1 = sc.seed_path([1], m)
        assert o0 == list(range(1, m + 1)) and d0 == 0 and s0 == sc.greedy_swaps(m - 1)
        assert o1 == [m] + list(range(1, m)) and d1 == 1
        assert s1 == [i + 1 for i in sc.greedy_swaps(m - 1)]
    assert sc.seed_path([0], 3) == ([1, 2, 3], 0, [1])
    assert sc.seed_path([1], 3) == ([3, 1, 2], 1, [2])
    assert sc.seed_path([1, 0], 4) == ([4, 1, 2, 3], 1, [2])
    # per-worker schedule length 2^(m-b) - (m-b) - 1
    assert len(sc.seed_path([0, 1, 1], 10)[2]) == 120


def test_alg2_joint_coverage_and_printed_bit_convention():
    """Union over workers covers all nonempty-parent models;
    the printed "prepend if bit == 0" does not (G9 / SURVEY V10)."""
    for m in range(4, 9):
        for b in range(1, m - 1):
            seen = set()
            for bits in itertools.product([0, 1], repeat=b):
                seen |= sc.worker_models(list(bits), m)
            assert len(seen) == sc.total_models(m)
    m, b = 8, 3
    seen = set()
    for bits in itertools.product([0, 1], repeat=b):
        flipped = [1 - x for x in bits]
        o, d, s = sc.seed_path(flipped, m)       # prepend on 0 == flip the bits
        s = [sum(bits) + t for t in sc.greedy_swaps(m - b)]   # printed d = sum(P_id)
        for p in sc.walk(m, s, start=o):
            seen |= sc.models_of_permutation(p)
    assert len(seen) < sc.total_models(m)


@pytest.mark.parametrize("m", [3, 5, 7, 9])
def test_exactly_once_ownership(m):
    """Reading G11: seed prefixes d..d+k plus each swap's new prefix
    set partition ALL m 2^(m-1) families (empty set included), no duplicates."""
    allf = sc.all_families(m)
    for b in range(0, m - 1):
        fams = []
        for bits in itertools.product([0, 1], repeat=b):
            own = sc.worker_owned_families(list(bits), m)
            # every family owned by beta has S n P = F_beta
            o, d, _ = sc.seed_path(list(bits), m)
            F = set(o[:d])
            P = set(range(m - b + 1, m + 1))
            assert all(set(S) & P == F for _, S in own)
            assert len(own) == 2 ** (m - b - 1) * (2 * (m - d) - (m - b))
            fams += own
        assert len(fams) == len(set(fams)) == len(allf)
        assert set(fams) == allf
