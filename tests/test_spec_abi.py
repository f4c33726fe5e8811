"""CPU: libtts's host-side speculative-beam-extension decisions (C-ABI,
host only) against the oracle's (oracle/spec.py, pinned in
test_oracle_spec.py): SelectSpec binning + greedy fill, DuplicateThenTruncate."""
import random

import pytest

from oracle.select import select_survivors
from oracle.spec import bin_score, select_spec, spec_plan


@pytest.fixture(scope="module")
def T():
    from paper_2509_00195_b200 import build, tts
    build.build()
    tts.load()
    return tts


@pytest.mark.parametrize("seed", range(40))
def test_spec_select_equals_oracle(T, seed):
    rnd = random.Random(seed)
    B = rnd.choice([1, 2, 4, 8])
    cand = sorted(rnd.sample(range(64), rnd.randint(1, 10)))
    last = [rnd.choice([0.0, 0.25, 0.5, 0.75, 1.0, rnd.random(), float("nan")]) for _ in cand]
    have = [rnd.randint(0, bin_score(s, B)[1] - 1) for s in last]
    free = rnd.randint(0, 20)
    got = T.spec_select(cand, last, have, free, B)
    want = dict(select_spec([(b, bin_score(s, B)[1], h) for b, s, h in zip(cand, last, have)], free))
    assert got == [want.get(b, 0) for b in cand]


@pytest.mark.parametrize("seed", range(40))
def test_spec_plan_equals_oracle(T, seed):
    rnd = random.Random(100 + seed)
    M = rnd.choice([1, 2, 4])
    N = M * rnd.randint(1, 6)
    scores = [rnd.randint(0, 4) / 4 for _ in range(N)]
    _, parent = select_survivors(scores, M)
    branches = [(rnd.randrange(N), rnd.randint(0, 40)) for _ in range(rnd.randint(0, N - 1))]
    lens = [rnd.randint(1, 300) for _ in range(N)]
    frac = [rnd.random() for _ in range(N)]
    nxt = [rnd.randint(1, 50) for _ in range(N)] if seed % 2 else None
    assert T.spec_plan(parent, M, branches, lens, frac, nxt) == tuple(map(list, spec_plan(parent, M, branches, lens,
                                                                                         frac, nxt)))
