"""The paper's combinatorics, written out plainly -- TEST INFRASTRUCTURE ONLY.

Independent of the product's host plan (paper_1901_07643_b200/csrc/plan.h); the
tests compare the two.  Positions and variables are 1-based here, as in the
paper.  Each function cites the passage it follows; the readings (G-numbers)
are listed in DESIGN.md.
"""
from __future__ import annotations

from itertools import combinations


def greedy_swaps(m: int) -> list[int]:
    """Alg.1 GreedySwaps(m) with the +1 of Eq.10.

    Upsilon(2) = [1];  Upsilon(m) = Upsilon(m-1) : [m-1, ..., 1] : [i+1 | i in Upsilon(m-1)].
    Reading G2: Alg.1's third segment as printed lacks the +1
    that PAPER.md:158 (step 3) and Eq.10 state; the +1 version is used.
    m = 1 has no swaps (|Upsilon(1)| = 2^1 - 1 - 1 = 0, Eq.9).
    """
    if m <= 1:
        return []
    if m == 2:
        return [1]
    prev = greedy_swaps(m - 1)
    return prev + list(range(m - 1, 0, -1)) + [i + 1 for i in prev]


def greedy_swaps_as_printed(m: int) -> list[int]:
    """Alg.1 exactly as printed at PAPER.md:170 (third segment NOT shifted).
    Kept only so a test can show it fails coverage."""
    if m == 2:
        return [1]
    prev = greedy_swaps_as_printed(m - 1)
    return prev + list(range(m - 1, 0, -1)) + [i for i in prev]


def schedule_length(m: int) -> int:
    """Eq.9 / Eq.12: |Upsilon(m)| = 2^m - 1 - m."""
    return 2 ** m - 1 - m


def apply_swap(order: list, i: int) -> list:
    """GRC_i's effect on the variable order (§1.3): transpose the
    variables at positions i and i+1 (1-based)."""
    o = list(order)
    o[i - 1], o[i] = o[i], o[i - 1]
    return o


def models_of_permutation(order) -> set:
    """Eq.5: the QRD of an order serves every family
    (order[j] | {order[1..k]}) with 1 <= k < j <= m -- m(m-1)/2 families.
    A family is (child, frozenset(parents))."""
    m = len(order)
    out = set()
    for k in range(1, m):
        pre = frozenset(order[:k])
        for j in range(k, m):
            out.add((order[j], pre))
    return out


def walk(m: int, schedule, start=None):
    """The permutations visited by replaying `schedule` from `start`
    (identity by default), as in Eq.7/Eq.8."""
    order = list(start) if start is not None else list(range(1, m + 1))
    perms = [order]
    for i in schedule:
        order = apply_swap(order, i)
        perms.append(order)
    return perms


def cumulative_model_counts(m: int, schedule) -> list[int]:
    """Number of distinct models solvable after each permutation of the walk
    (the counts printed beside Eq.8)."""
    seen = set()
    counts = []
    for p in walk(m, schedule):
        seen |= models_of_permutation(p)
        counts.append(len(seen))
    return counts


def new_models_after_swap(order_after, i: int, seen: set) -> set:
    """SPEC.md:150-158 / §3 greedy choice: after a swap at i only
    the length-i prefix set changes, so the new models are those with parent
    set set(order[1..i]) and a child after position i that are not yet seen."""
    pre = frozenset(order_after[:i])
    return {(c, pre) for c in order_after[i:] if (c, pre) not in seen}


def verify_coverage(m: int, schedule) -> int:
    """Distinct nonempty-parent models covered by the walk;
    complete iff it equals m(2^(m-1) - 1)."""
    seen = set()
    for p in walk(m, schedule):
        seen |= models_of_permutation(p)
    return len(seen)


def total_models(m: int) -> int:
    """m(2^(m-1) - 1) nonempty-parent families."""
    return m * (2 ** (m - 1) - 1)


def rotation_flops(m: int, schedule) -> int:
    """Sum over the schedule of the per-GRC cost 6(m - i + 1)."""
    return sum(6 * (m - i + 1) for i in schedule)


def predicted_rotation_flops(m: int) -> int:
    """Eq.13 closed form, read with G6 ("62^m" = 6*2^m):
    T(m) = 3m 2^m + 6 2^m - 3m^2 - 9m - 6."""
    return 3 * m * 2 ** m + 6 * 2 ** m - 3 * m * m - 9 * m - 6


def runtime_recurrence(m: int) -> int:
    """Eq.11 evaluated literally with Eq.12 for |Upsilon|:
    T(m) = [T(m-1) + 6|Upsilon(m-1)|] + sum_{i=1}^{m-1} 6(m-i+1) + T(m-1), T(2)=12
    (T(2) = one GRC at i=1 on a 2-column factor, 6(2-1+1) = 12)."""
    if m == 2:
        return 12
    t = runtime_recurrence(m - 1)
    return (t + 6 * schedule_length(m - 1)) + sum(6 * (m - i + 1) for i in range(1, m)) + t


def seed_path(bits, m: int):
    """Alg.2 SeedPathCalculator(P_id, m) with readings
    G7 (loop to m, not n), G8 (k = m - len(P_id)), G9 (prepend when the bit is
    1 -- as printed, "== 0", it fails coverage) and G10
    (Upsilon = d + GreedySwaps(k) elementwise; needs k >= 2).
    bits: the processor's binary array P_id (P_id[m - i] selects variable i).
    Returns (seed order upsilon, d, shifted schedule)."""
    b = len(bits)
    k = m - b
    if k < 2:
        raise ValueError("Alg.2 needs k = m - len(P_id) >= 2")
    order = list(range(1, k + 1))
    for i in range(k + 1, m + 1):
        if bits[m - i] == 1:
            order.insert(0, i)
        else:
            order.append(i)
    d = sum(bits)
    return order, d, [d + s for s in greedy_swaps(k)]


def worker_models(bits, m: int) -> set:
    """All models of all permutations a worker visits."""
    order, d, sched = seed_path(bits, m)
    seen = set()
    for p in walk(m, sched, start=order):
        seen |= models_of_permutation(p)
    return seen


def worker_owned_families(bits, m: int) -> list:
    """Exactly-once ownership (reading G11 / SURVEY.md V11): worker beta keeps
    (a) its seed prefixes of sizes d..d+k (size 0 = the empty set, only when
    d = 0; size m has no child) and (b) each swap's new prefix set, with every
    child after the prefix.  Returns a list (duplicates would show)."""
    order, d, sched = seed_path(bits, m)
    k = m - len(bits)
    out = []
    for size in range(d, d + k + 1):
        pre = frozenset(order[:size])
        out += [(c, pre) for c in order[size:]]
    for p, i in zip(walk(m, sched, start=order)[1:], sched):
        pre = frozenset(p[:i])
        out += [(c, pre) for c in p[i:]]
    return out


def all_families(m: int) -> set:
    """Every (child, parent set) including the empty set: m 2^(m-1)."""
    out = set()
    for c in range(1, m + 1):
        others = [u for u in range(1, m + 1) if u != c]
        for r in range(0, m):
            for s in combinations(others, r):
                out.add((c, frozenset(s)))
    return out
