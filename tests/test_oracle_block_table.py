"""Pins for oracle.block_table / oracle.run (CPU): the hand-derived C1 trace of
SURVEY.md 8(c), its copy-on-write variant, and the paper's invariants checked
at every fork of randomised small runs."""
import os
import random

import numpy as np
import pytest

from oracle.block_table import BlockTableSim, OutOfPages
from oracle.run import OracleRun
from synth import workload

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _c1_sim(step1_len):
    sim = BlockTableSim(num_pages=16, P=16)
    sim.init_request(0, 4, 32)
    for _ in range(step1_len):
        sim.append([0], [[1, 1, 1, 1]])
    return sim


def _live(sim, lo=0, hi=None):
    return {p: r for p, r in enumerate(sim.ref) if r and p >= lo and (hi is None or p < hi)}


def test_c1_hand_trace():
    """tests/golden/c1_trace.txt (derived under rules C2-C8)."""
    sim = _c1_sim(16)
    assert sim.tables[0] == [[0, 1, 2], [0, 1, 3], [0, 1, 4], [0, 1, 5]]
    sim.fork([0], [[0.9, 0.1, 0.5, 0.5]], 2)
    assert sim.tables[0] == [[0, 1, 2], [0, 1, 2], [0, 1, 4], [0, 1, 4]]
    assert _live(sim) == {0: 4, 1: 4, 2: 2, 4: 2}
    assert [p for p in sim.free_set() if p < 6] == [3, 5]
    for _ in range(16):
        sim.append([0], [[1, 1, 1, 1]])
    assert sim.tables[0] == [[0, 1, 2, 3], [0, 1, 2, 5], [0, 1, 4, 6], [0, 1, 4, 7]]
    sim.fork([0], [[0.5, 0.75, 0.75, 0.75]], 2)  # three-way tie, beam 3 loses
    assert sim.tables[0] == [[0, 1, 2, 5], [0, 1, 2, 5], [0, 1, 4, 6], [0, 1, 4, 6]]
    assert _live(sim) == {0: 4, 1: 4, 2: 2, 4: 2, 5: 2, 6: 2}
    assert [p for p in sim.free_set() if p < 8] == [3, 7]
    for _ in range(16):
        sim.append([0], [[1, 1, 1, 1]])
    assert sim.tables[0] == [[0, 1, 2, 5, 3], [0, 1, 2, 5, 7], [0, 1, 4, 6, 8], [0, 1, 4, 6, 9]]
    assert sim.lens[0] == [80] * 4


def test_c1_golden_file_matches():
    with open(os.path.join(GOLDEN, "c1_trace.txt")) as f:
        rows = [ln.split("#")[0].strip() for ln in f]
    rows = [r for r in rows if r]
    sim = _c1_sim(16)
    got = [" ".join(map(str, sum(sim.tables[0], [])))]
    sim.fork([0], [[0.9, 0.1, 0.5, 0.5]], 2)
    got.append(" ".join(map(str, sum(sim.tables[0], []))))
    for _ in range(16):
        sim.append([0], [[1, 1, 1, 1]])
    got.append(" ".join(map(str, sum(sim.tables[0], []))))
    sim.fork([0], [[0.5, 0.75, 0.75, 0.75]], 2)
    got.append(" ".join(map(str, sum(sim.tables[0], []))))
    for _ in range(16):
        sim.append([0], [[1, 1, 1, 1]])
    got.append(" ".join(map(str, sum(sim.tables[0], []))))
    assert got == rows


def test_c1_cow_variant():
    """Step 1 of 10 tokens: the fork frees {3,5} and re-allocates them as CoW
    copies; page ids equal the pre-fork ids but the contents differ."""
    sim = _c1_sim(10)
    before = {p: list(sim.content[p]) for p in (2, 3, 4, 5)}
    sim.fork([0], [[0.9, 0.1, 0.5, 0.5]], 2)
    assert sim.tables[0] == [[0, 1, 2], [0, 1, 3], [0, 1, 4], [0, 1, 5]]
    assert all(sim.ref[p] == 1 for p in (2, 3, 4, 5))
    assert sim.content[3][:10] == before[2][:10]   # copy of beam 0's page
    assert sim.content[5][:10] == before[4][:10]   # copy of beam 2's page
    assert sim.content[3][:10] != before[3][:10]
    assert sim.gather(0, 1) == sim.gather(0, 0)


def test_partial_prompt_cow_at_install():
    sim = BlockTableSim(num_pages=32, P=16)
    sim.init_request(0, 4, 37)  # pages 0,1,2 (2 partial) ; copies 3,4,5
    assert sim.tables[0] == [[0, 1, 2], [0, 1, 3], [0, 1, 4], [0, 1, 5]]
    assert sim.ref[:6] == [4, 4, 1, 1, 1, 1]
    assert all(sim.gather(0, b) == sim.gather(0, 0) for b in range(4))


def test_out_of_pages():
    sim = BlockTableSim(num_pages=3, P=16)
    sim.init_request(0, 2, 32)
    sim.append([0], [[1, 0]])
    with pytest.raises(OutOfPages):
        sim.append([0], [[0, 1]])


def _check_invariants(run: OracleRun, rec):
    sim, c = run.sim, run.cfg
    P = c.P
    counts = {}
    total_pages = 0
    for r, rows in sim.tables.items():
        assert len(rows) == c.N                                  # beam count stays N
        for b, row in enumerate(rows):
            n = sim.lens[r][b]
            assert len(row) == -(-n // P)
            total_pages += len(row)
            assert len(set(row)) == len(row)
            for p in row:
                counts[p] = counts.get(p, 0) + 1
                assert not sim.is_free[p]                        # no table -> free page
            if n % P:
                assert sim.ref[row[-1]] == 1                     # C6 invariant
    assert sum(sim.ref) == total_pages                           # refcount conservation
    for p in range(sim.num_pages):
        assert sim.ref[p] == counts.get(p, 0)                    # C8 definition
        assert sim.is_free[p] == (sim.ref[p] == 0)               # free U used = pool
    for r in rec.reqs:
        rows = sim.tables[r]
        # children of one parent hold the parent's logical sequence:
        # siblings read identical token sequences through their tables
        for cc in range(c.N):
            first = (cc // c.M) * c.M
            assert rec.parents[r][cc] == rec.parents[r][first]
            assert sim.gather(r, cc) == sim.gather(r, first)
        # DFS contiguity (ledger C5): beams sharing a page form a contiguous range
        where = {}
        for b, row in enumerate(rows):
            for i, p in enumerate(row):
                where.setdefault(p, []).append(b)
        for p, bs in where.items():
            assert bs == list(range(bs[0], bs[0] + len(bs)))
            if len(bs) > 1:
                # shared pages are full
                i = rows[bs[0]].index(p)
                assert all(sim.lens[r][b] >= (i + 1) * P for b in bs)
        # prefix closure and LCP(pages) == floor(LCP(tokens)/P)
        for b in range(c.N - 1):
            a_row, b_row = rows[b], rows[b + 1]
            k = 0
            while k < min(len(a_row), len(b_row)) and a_row[k] == b_row[k]:
                k += 1
            assert all(a_row[i] != b_row[i] for i in range(k, min(len(a_row), len(b_row))))
            la, lb = run.lists[r][b], run.lists[r][b + 1]
            t = 0
            while t < min(len(la), len(lb)) and (la[t] == lb[t]).all():
                t += 1
            lcp_tokens = c.prompt + t
            assert k == lcp_tokens // P


@pytest.mark.parametrize("seed", range(12))
def test_random_runs_invariants(seed):
    rnd = random.Random(seed)
    N = rnd.choice([4, 8, 16])
    M = rnd.choice([m for m in (2, 4, 8) if N % m == 0])
    cfg = workload.Config(f"rand{seed}", R=rnd.choice([1, 2, 3]), N=N, M=M, L=1, Hq=2, Hkv=1, d=8,
                          P=rnd.choice([4, 16]), prompt=rnd.choice([0, 5, 16, 37]), n_steps=5,
                          step_len=0, ln_mu=np.log(rnd.choice([3, 8, 20])), ln_sigma=1.0, ln_cap=40,
                          seed=1000 + seed)
    run = OracleRun(cfg)
    n_forks = []
    run.run(on_fork=lambda rr, rec: (_check_invariants(rr, rec), n_forks.extend(rec.reqs)))
    assert len(n_forks) == cfg.R * (cfg.n_steps - 1)


def test_stats_unique_logical():
    sim = _c1_sim(16)
    sim.fork([0], [[0.9, 0.1, 0.5, 0.5]], 2)
    sim.append([0], [[1, 1, 1, 1]])
    u, lg = sim.stats([0], [[1, 1, 1, 1]])
    # pages 0,1 (32), 2 and 4 (16 each), four new private pages with 1 token
    assert u == 32 + 32 + 4 and lg == 4 * 49
