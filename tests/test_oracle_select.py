"""Pins for oracle.select (CPU).  Each check is independent of order_key."""
import itertools
import math
import random

import numpy as np
import pytest

from oracle.select import SelectError, select_survivors


def beats(a, ia, b, ib):
    """a (index ia) ranks ahead of b (index ib): SURVEY ledger C3/C4, written
    with Python float comparisons (where -0.0 == 0.0 already holds)."""
    na, nb = math.isnan(a), math.isnan(b)
    if na and nb:
        return ia < ib
    if na != nb:
        return nb
    if a != b:
        return a > b
    return ia < ib


def brute_force(scores, M):
    N = len(scores)
    K = N // M
    found = []
    for sub in itertools.combinations(range(N), K):
        s = set(sub)
        if all(beats(scores[i], i, scores[j], j) for i in s for j in range(N) if j not in s):
            found.append(sorted(sub))
    assert len(found) == 1  # strict total order -> unique correct subset
    return found[0]


def test_spec_worked_example():
    # BeamSearch n=4, B=2, [0.9, 0.1, 0.5, 0.5] -> {0, 2}
    surv, parent = select_survivors([0.9, 0.1, 0.5, 0.5], 2)
    assert surv == [0, 2]
    assert parent == [0, 0, 2, 2]


def test_all_equal_lowest_ids():
    # SPEC S:48 (n = B -> single lowest-id beam), generalised to any K
    assert select_survivors([0.3] * 4, 4)[0] == [0]
    assert select_survivors([0.3] * 12, 3)[0] == [0, 1, 2, 3]


@pytest.mark.parametrize("seed", range(40))
def test_brute_force_small(seed):
    rnd = random.Random(seed)
    N = rnd.choice([2, 4, 6, 8, 9, 10, 12])
    Ms = [m for m in range(1, N + 1) if N % m == 0]
    M = rnd.choice(Ms)
    pool = [0.0, -0.0, 0.25, 0.5, 1.0, float("nan"), float("inf"), float("-inf"), 0.75]
    scores = [rnd.choice(pool) if rnd.random() < 0.6 else rnd.random() for _ in range(N)]
    surv, parent = select_survivors(scores, M)
    assert surv == brute_force(scores, M)
    assert parent == [surv[c // M] for c in range(N)]


@pytest.mark.parametrize("seed", range(10))
def test_library_sort(seed):
    rs = np.random.RandomState(seed)
    N, M = 512, 8
    scores = (rs.randint(0, 64, size=N) / 64.0).astype(np.float32)
    ref = sorted(np.lexsort((np.arange(N), -scores.astype(np.float64)))[: N // M].tolist())
    assert select_survivors(scores.tolist(), M)[0] == ref


def test_nan_and_signed_zero():
    s = [float("nan"), -0.0, 0.0, float("-inf")]
    assert select_survivors(s, 2)[0] == [1, 2]        # -0 == +0, tie by index
    assert select_survivors(s, 4)[0] == [1]
    s = [float("nan"), float("nan"), float("-inf"), float("nan")]
    assert select_survivors(s, 2)[0] == [0, 2]        # -inf beats NaN; NaNs by index
    assert select_survivors([float("nan")] * 4, 2)[0] == [0, 1]
    assert select_survivors([2.0, float("inf"), 5.0, -3.0], 2)[0] == [1, 2]


@pytest.mark.parametrize("seed", range(10))
def test_invariants(seed):
    rnd = random.Random(seed)
    N, M = 64, 4
    scores = [rnd.randint(0, 15) / 16 for _ in range(N)]
    surv, parent = select_survivors(scores, M)
    # sum of branch counts == N
    assert len(parent) == N and all(parent.count(s) == M for s in surv)
    # the kept set depends only on the (id, score) pairs: shuffling
    # the pairs and re-sorting by (score desc, id asc) keeps the same ids
    pairs = list(enumerate(scores))
    rnd.shuffle(pairs)
    keyed = sorted(pairs, key=lambda p: (-p[1], p[0]))[: N // M]
    assert sorted(i for i, _ in keyed) == surv
    # monotonicity
    for b in surv:
        s2 = list(scores)
        s2[b] = s2[b] + 0.5
        assert b in select_survivors(s2, M)[0]


def test_errors():
    with pytest.raises(SelectError):
        select_survivors([], 2)
    with pytest.raises(SelectError):
        select_survivors([0.1, 0.2, 0.3], 2)


# ---------------------------------------------------------------------------
# Selection variants: diverse selection and dynamic branching
from oracle.select import (POLICY_DIVERSE, POLICY_DYNAMIC, POLICY_TOPK, branch_counts_dynamic,  # noqa: E402
                           select_diverse, select_dynamic, select_policy)


def test_dynamic_spec_worked_example():
    # DynamicBranching, n = 8, scores [0.8, 0.2] -> branch counts [6, 2]
    assert branch_counts_dynamic([0.8, 0.2], 8) == [6, 2]
    surv, counts, parent = select_dynamic([0.8, 0.2], 1)  # both beams kept (K = N / 1), N = 2
    assert surv == [0, 1] and counts == [1, 1]


def _lr_brute(q_plus_one, N):
    """All integer vectors c >= 1 with sum N; the ones closest to the quotas
    (L1), lowest-index preference among ties (lexicographically largest)."""
    K = len(q_plus_one)
    best, arg = None, []
    for c in itertools.product(range(1, N + 1), repeat=K):
        if sum(c) != N:
            continue
        d = sum(abs(ci - ti) for ci, ti in zip(c, q_plus_one))
        if best is None or d < best - 1e-12:
            best, arg = d, [list(c)]
        elif abs(d - best) <= 1e-12:
            arg.append(list(c))
    return best, arg


@pytest.mark.parametrize("seed", range(60))
def test_dynamic_counts_exhaustive(seed):
    """The largest-remainder counts minimise the L1 distance to the quotas
    1 + q_i over every apportionment with a floor of one and the exact sum
    ("exhaustive apportionment check"); each count is within one
    of its quota; ties go to the lower survivor index."""
    rnd = random.Random(seed)
    K = rnd.randint(1, 4)
    N = K + rnd.randint(0, 7)
    sc = [rnd.choice([0.0, 0.25, 0.5, 0.8, 0.2, rnd.random()]) for _ in range(K)]
    c = branch_counts_dynamic(sc, N)
    assert sum(c) == N and min(c) >= 1
    W = sum(sc) or None
    t = [1 + ((N - K) * s / W if W else (N - K) / K) for s in sc]
    assert all(abs(ci - ti) < 1 for ci, ti in zip(c, t))
    best, arg = _lr_brute(t, N)
    d = sum(abs(ci - ti) for ci, ti in zip(c, t))
    assert abs(d - best) <= 1e-12
    assert c == max(arg)  # lexicographically largest = extra children to lower indices first


def test_dynamic_special_cases():
    assert branch_counts_dynamic([0.5, 0.5, 0.5, 0.5], 8) == [2, 2, 2, 2]      # equal scores: equal split
    assert branch_counts_dynamic([0.0, 0.0], 5) == [3, 2]                      # all zero: equal weights
    assert branch_counts_dynamic([float("nan"), 1.0], 6) == [1, 5]            # NaN weighs 0, floor 1
    assert branch_counts_dynamic([1.0], 7) == [7]


def test_diverse_brute_force_and_structure():
    rnd = random.Random(5)
    for _ in range(200):
        B = rnd.choice([1, 2, 4, 8])
        n = rnd.choice([1, 2, 4])
        N = B * n
        sc = [rnd.randint(0, 4) / 4 for _ in range(N)]
        surv, parent = select_diverse(sc, B)
        for s in range(B):
            sub = list(range(s * n, (s + 1) * n))
            # the survivor of subtree s beats every other beam of it (brute force)
            assert surv[s] in sub
            assert all(beats(sc[surv[s]], surv[s], sc[j], j) for j in sub if j != surv[s])
            # its n children form subtree s again
            assert parent[s * n:(s + 1) * n] == [surv[s]] * n
    assert select_diverse([0.1, 0.9, 0.3, 0.3], 4)[1] == [0, 1, 2, 3]          # B = N: identity
    assert select_diverse([0.1, 0.9, 0.3, 0.3], 1)[1] == [1, 1, 1, 1]          # B = 1: global top-1
    assert select_diverse([0.3] * 8, 2)[0] == [0, 4]                           # ties: lowest index


def test_policy_dispatch_and_topk_equivalence():
    sc = [0.9, 0.1, 0.5, 0.5]
    assert select_policy(sc, POLICY_TOPK, 2) == [0, 0, 2, 2]
    assert select_policy(sc, POLICY_DIVERSE, 2) == [0, 0, 2, 2]
    # survivors {0, 2} (0.9, 0.5): quotas 2 x [0.9, 0.5] / 1.4 = [1.29, 0.71] -> [2, 1] + the
    # remaining child to the larger fraction (0.71) -> [2, 2]
    assert select_policy(sc, POLICY_DYNAMIC, 2) == [0, 0, 2, 2]
    # survivors {0, 2} (0.9, 0.3): quotas [1.5, 0.5] -> [2, 1], equal fractions -> lower index -> [3, 1]
    assert select_policy([0.9, 0.1, 0.3, 0.3], POLICY_DYNAMIC, 2) == [0, 0, 0, 2]
    # beam search is dynamic branching with a uniform count: fork_parents == fork
    from oracle.block_table import BlockTableSim
    a, b = BlockTableSim(64, 16), BlockTableSim(64, 16)
    for sim in (a, b):
        sim.init_request(0, 4, 37)
        for _ in range(21):
            sim.append([0], [[1, 1, 1, 1]])
    a.fork([0], [sc], 2)
    b.fork_parents([0], [select_policy(sc, POLICY_TOPK, 2)])
    assert a.tables == b.tables and a.ref == b.ref and a.lens == b.lens
