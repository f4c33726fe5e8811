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
