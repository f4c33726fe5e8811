"""Pins for oracle.spec (CPU): Speculative Beam Extension, decode side
(Alg. 1, binning P:316-322, DuplicateThenTruncate
P:310-311) against SPEC S:240-257's worked examples and the paper's
algorithmic-equivalence property."""
import math
import random

import numpy as np
import pytest

from oracle.block_table import BlockTableSim
from oracle.select import select_survivors
from oracle.spec import SpecRun, SpecSim, bin_score, select_spec, spec_plan
from synth import workload


def test_bin_score_spec_examples():
    assert bin_score(0.9, 4) == (1, 4)      # S:244 B=4, 0.9 -> j=1, M=4
    assert bin_score(0.37, 1) == (1, 1)     # S:245 B=1 -> j=1, M=1
    assert bin_score(0.0, 4) == (4, 1)      # S:246 lowest bin, M=1
    assert bin_score(0.75, 4) == (1, 4)     # boundary -> the higher bin
    assert bin_score(0.5, 4) == (2, 3)
    assert bin_score(1.0, 8) == (1, 8)
    assert bin_score(float("nan"), 4) == (4, 1)


def test_select_spec_spec_examples():
    assert select_spec([(0, 4, 0), (1, 2, 0)], 5) == [(0, 4), (1, 1)]
    assert select_spec([(0, 4, 0), (1, 2, 0)], 0) == []
    assert select_spec([(7, 3, 0)], 10) == [(7, 3)]                     # S:252 potential caps
    assert select_spec([(3, 2, 0), (1, 2, 0), (2, 4, 3)], 3) == [(2, 1), (1, 2)]  # M desc, then lower id; caps


@pytest.mark.parametrize("seed", range(30))
def test_select_spec_priority_property(seed):
    rnd = random.Random(seed)
    cand = [(b, rnd.randint(1, 4), 0) for b in rnd.sample(range(20), rnd.randint(1, 8))]
    cand = [(b, m, rnd.randint(0, m - 1)) for b, m, _ in cand]
    free = rnd.randint(0, 12)
    out = dict(select_spec(cand, free))
    assert sum(out.values()) == min(free, sum(m - k for _, m, k in cand))
    for b, m, k in cand:
        assert out.get(b, 0) <= m - k
        for b2, m2, k2 in cand:  # no smaller-M beam gets a branch while a larger-M one has unmet cap
            if m2 > m and out.get(b2, 0) < m2 - k2:
                assert out.get(b, 0) == 0


def test_duplicate_then_truncate_spec_examples():
    # S:56-58, M = 2: one survivor (beam 0) with one branch of 100 speculative tokens
    parent = [0, 0]
    assert spec_plan(parent, 2, [], [40, 7], [0.3, 0.3])[1] == [40, 40]            # no speculative tokens
    pr, nl, h = spec_plan(parent, 2, [(0, 100), (0, 100)], [40, 7], [1.0, 1.0])    # R = 1, sigma = 0
    assert h == [100, 100] and nl == [140, 140] and pr == [2, 3]
    pr, nl, h = spec_plan(parent, 2, [(0, 100), (0, 100)], [40, 7], [0.85, 0.85])  # R = 0.85, sigma = 0
    assert h == [100, 85]
    pr, nl, h = spec_plan(parent, 2, [(0, 100)], [40, 7], [0.85, 0.85])            # one branch: the duplicate
    assert pr == [2, 0] and h == [100, 0] and nl == [140, 40]
    assert spec_plan(parent, 2, [(0, 100)], [40, 7], [0.5, 0.5], next_len=[30, 30])[2] == [30, 0]  # capped


def test_branch_and_truncate_tables():
    P = 16
    sim = SpecSim(64, P)
    sim.init_request(0, 2, 20, [("p", 0, i) for i in range(20)])
    for t in range(5):
        sim.append([0], [[1, 1]], [[("d", 0, t, b) for b in range(2)]])
    # beam 0 (25 tokens, partial page) gets two branches: each copies the partial page
    rows = sim.branch(0, [0, 0])
    assert rows == [2, 3]
    assert sim.tables[0][2][0] == sim.tables[0][0][0] and sim.tables[0][2][1] != sim.tables[0][0][1]
    for t in range(5, 25):
        sim.append([0], [[0, 0, 1, 1]], [[("d", 0, t, b) for b in range(4)]])
    assert sim.lens[0] == [25, 25, 45, 45]
    # children: branch 2 kept whole, branch 3 truncated to 10 tokens, then a duplicate of beam 0
    sim.fork_trunc(0, [2, 3, 0], [45, 35, 25])
    assert sim.lens[0] == [45, 35, 25]
    assert sim.gather(0, 1)[:25] == sim.gather(0, 2) and len(sim.gather(0, 1)) == 35
    used = {p for row in sim.tables[0] for p in row}
    assert all(sim.ref[p] == sum(row.count(p) for row in sim.tables[0]) for p in used)
    assert all(sim.ref[p] == 0 for p in range(64) if p not in used)


def test_spec_worked_example_occupancy():
    """two beams with step lengths 10 and 100 and two slots: beam A
    finishes at token 10, one speculative branch of A fills the free slot for
    tokens 11-100 -> occupancy 2/2 for all 100 ticks vs 1.1/2 without."""
    cfg = workload.Config("spec-ex", R=1, N=2, M=1, L=1, Hq=2, Hkv=1, d=16, P=16, prompt=16, n_steps=2,
                          step_len=0, seed=5)
    lens = np.array([[[3, 3], [10, 100]]])
    on = SpecRun(cfg, True, lengths=lens, scores_fn=lambda r, s: [0.9, 0.2]).run()
    off = SpecRun(cfg, False, lengths=lens, scores_fn=lambda r, s: [0.9, 0.2]).run()
    assert on.running[3:] == [2] * 100
    assert sum(off.running[3:]) / 100 == pytest.approx(1.1)
    assert on.forks[0]["parent"] == off.forks[0]["parent"]


@pytest.mark.parametrize("seed", range(8))
def test_speculation_is_algorithmically_equivalent(seed):
    """speculation on and off select the same survivors at
    every fork (same scores, same inputs); every child's token sequence starts
    with its parent's; the running rows never exceed the N slots; head starts
    never lengthen a run."""
    rnd = random.Random(seed)
    N, M = rnd.choice([(4, 2), (8, 2), (8, 4), (16, 4)])
    cfg = workload.Config(f"spec{seed}", R=rnd.choice([1, 2]), N=N, M=M, L=1, Hq=4, Hkv=2, d=16, P=16,
                          prompt=rnd.choice([0, 5, 32]), n_steps=4, step_len=0, ln_mu=math.log(12),
                          ln_sigma=1.0, ln_cap=60, seed=700 + seed)
    on = SpecRun(cfg, True).run()
    off = SpecRun(cfg, False).run()
    assert [f["parent"] for f in on.forks] == [f["parent"] for f in off.forks]
    assert on.beam_steps <= off.beam_steps and on.iterations <= off.iterations
    assert all(r <= c for r, c in zip(on.running, on.capacity))
    assert sum(on.running) / sum(on.capacity) >= sum(off.running) / sum(off.capacity) - 1e-12
    for f in on.forks:
        for c, (pr, nl) in enumerate(zip(f["parent_rows"], f["new_lens"])):
            assert nl >= 0
        used = {p for row in f["tables"] for p in row}
        assert all(f["ref"][p] >= 1 for p in used)
        assert set(f["free"]).isdisjoint(used)
