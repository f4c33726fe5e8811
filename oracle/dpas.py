"""Dynamic Prefix-Aware Scheduling under a memory budget (oracle; test
infrastructure only).  PAPER.md 4.2 and Appendix A.

A CoT is a beam's context as a path of nodes (here: KV pages, root first; the
paper's nodes are beams/steps -- pages are this build's unit, DESIGN.md
ledger C30).  P(a, b) = the number of common leading nodes (shared prefix).
* greedy schedule: order[0] = the first CoT in input order; then repeatedly
  the unscheduled CoT maximising P with its predecessor, ties to input order
  ("T_{k+1} = argmax P(c_k, c_i)").
* tries: consecutive CoTs of the order are packed into one trie while the
  union of their nodes fits the budget (first fit, "the largest
  possible group of consecutively scheduled CoTs that can fit into memory";
  SPEC S:199).  A CoT larger than the budget is a trie by itself.
* cost = sum_i (Nodes(T_i) - P(T_i, T_{i+1})), P(T_i, T_{i+1}) = the nodes the
  two tries share, P(T_last, .) = 0.
"""
from __future__ import annotations

import itertools
from typing import List, Sequence, Tuple


def shared_prefix(a: Sequence, b: Sequence) -> int:
    n = 0
    for x, y in zip(a, b):
        if x != y:
            break
        n += 1
    return n


def greedy_schedule(cots: Sequence[Sequence]) -> List[int]:
    if not cots:
        raise ValueError("empty instance")
    order = [0]
    left = list(range(1, len(cots)))
    while left:
        prev = cots[order[-1]]
        best = max(left, key=lambda i: (shared_prefix(prev, cots[i]), -i))
        order.append(best)
        left.remove(best)
    return order


def prefix_sum(order: Sequence[int], cots: Sequence[Sequence]) -> int:
    return sum(shared_prefix(cots[order[k]], cots[order[k + 1]]) for k in range(len(order) - 1))


def brute_force_schedule(cots: Sequence[Sequence]) -> Tuple[List[int], int]:
    if len(cots) > 9:
        raise ValueError("oracle limit exceeded")
    best, arg = -1, None
    for perm in itertools.permutations(range(len(cots))):
        s = prefix_sum(perm, cots)
        if s > best:
            best, arg = s, list(perm)
    return arg, best


def is_locally_optimal(order: Sequence[int], cots: Sequence[Sequence]) -> bool:
    base = prefix_sum(order, cots)
    o = list(order)
    for i in range(len(o)):
        for j in range(i + 1, len(o)):
            o[i], o[j] = o[j], o[i]
            better = prefix_sum(o, cots) > base
            o[i], o[j] = o[j], o[i]
            if better:
                return False
    return True


def pack_tries(order: Sequence[int], cots: Sequence[Sequence], budget: int) -> List[List[int]]:
    """First-fit packing of consecutive CoTs into tries of <= budget nodes."""
    tries: List[List[int]] = []
    nodes: set = set()
    for i in order:
        path = set(cots[i])
        if tries and len(nodes | path) <= budget:
            tries[-1].append(i)
            nodes |= path
        else:
            tries.append([i])
            nodes = set(path)
    return tries


def eviction_cost(tries: Sequence[Sequence[int]], cots: Sequence[Sequence]) -> Tuple[int, int]:
    """(cost, shared) = (sum_i Nodes(T_i) - P(T_i, T_{i+1}), sum_i P(T_i, T_{i+1}))."""
    sets = [set().union(*[set(cots[i]) for i in t]) for t in tries]
    shared = sum(len(sets[k] & sets[k + 1]) for k in range(len(sets) - 1))
    return sum(len(s) for s in sets) - shared, shared
