"""Pins for oracle.dpas (CPU): Dynamic Prefix-Aware Scheduling (PAPER.md 4.2,
Appendix A) against SPEC S:150-199's worked examples, brute force, the
Appendix A local-optimality theorem and the cost identity; and, on beam
trees from the block-table simulator, the paper's implementation note
("grouping beams spawned from the same parent ... preserving the relative
order of the parent beams") = the explicit greedy."""
import random

import pytest

from oracle.block_table import BlockTableSim
from oracle.dpas import (brute_force_schedule, eviction_cost, greedy_schedule, is_locally_optimal, pack_tries,
                         prefix_sum, shared_prefix)

C1, C2, C3 = list("ABC"), list("ABD"), list("AE")


def test_spec_examples():
    cots = [C1, C2, C3]
    order = greedy_schedule(cots)
    assert order == [0, 1, 2] and prefix_sum(order, cots) == 3
    assert brute_force_schedule(cots)[1] == 3
    assert greedy_schedule([C1]) == [0] and prefix_sum([0], [C1]) == 0
    assert greedy_schedule([list("AB"), list("CD"), list("EF")]) == [0, 1, 2]  # S:155 disjoint -> input order
    tries = pack_tries(order, cots, 3)                                         # one CoT per trie (budget = 3 nodes)
    assert tries == [[0], [1], [2]] and eviction_cost(tries, cots) == (5, 3)  # S:162 (3-2)+(3-1)+(2-0)
    assert eviction_cost([[0]], [C1]) == (3, 0)
    assert eviction_cost([[0], [1]], [C1, C1]) == (3, 3)                       # S:164 identical CoTs
    assert shared_prefix(C1, C2) == 2 and shared_prefix(C1, C1) == 3 and shared_prefix(list("AB"), list("CD")) == 0
    assert not is_locally_optimal([0, 2, 1], cots)  # a worse order (score 2) is improved by a swap
    assert is_locally_optimal([0], [C1])


def _random_tree_cots(rnd, n):
    """CoTs from a random branching tree: each path extends a random earlier prefix."""
    cots = [[("r", 0)]]
    for k in range(1, n):
        base = rnd.choice(cots)
        cut = rnd.randint(0, len(base))
        cots.append(base[:cut] + [("n", k, j) for j in range(rnd.randint(1, 3))])
    rnd.shuffle(cots)
    return cots


@pytest.mark.parametrize("seed", range(100))
def test_local_optimality_theorem(seed):
    """Appendix A.2: no single swap improves the greedy schedule's score;
    greedy never beats brute force; cost + shared == sum of trie nodes."""
    rnd = random.Random(seed)
    cots = _random_tree_cots(rnd, rnd.randint(1, 8))
    g = greedy_schedule(cots)
    assert is_locally_optimal(g, cots)
    assert prefix_sum(g, cots) <= brute_force_schedule(cots)[1]
    budget = rnd.randint(1, 12)
    tries = pack_tries(g, cots, budget)
    cost, shared = eviction_cost(tries, cots)
    assert cost + shared == sum(len(set().union(*[set(cots[i]) for i in t])) for t in tries)
    assert sorted(sum(tries, [])) == sorted(g)
    for t in tries:
        assert len(t) == 1 or len(set().union(*[set(cots[i]) for i in t])) <= budget


@pytest.mark.parametrize("seed", range(10))
def test_parent_grouping_is_the_greedy_on_beam_trees(seed):
    """Beam trees of the block-table simulator (DFS order by ledger C5): the
    pages of the beams in index order are a greedy schedule."""
    rnd = random.Random(50 + seed)
    N, M = rnd.choice([(8, 2), (16, 4), (12, 3)])
    sim = BlockTableSim(4000, 16, track_content=False)
    sim.init_request(0, N, rnd.choice([0, 16, 37]))
    for step in range(4):
        for _ in range(rnd.randint(5, 40)):
            sim.append([0], [[rnd.random() < 0.9 for _ in range(N)]])
        sim.fork([0], [[rnd.randint(0, 4) / 4 for _ in range(N)]], M)
    cots = [list(row) for row in sim.tables[0]]
    assert prefix_sum(list(range(N)), cots) == prefix_sum(greedy_schedule(cots), cots)
    assert greedy_schedule(cots) == list(range(N))
