"""Beam selection by full sort (oracle; test infrastructure only).

PAPER.md 3.1: "standard Beam Search selects the top-K candidates
globally with a static branching factor".  With N live beams and branching
factor M, K = N / M survivors are kept (SPEC S:32 ``n mod B == 0``)
and each is replicated M times.

Order (SURVEY ledger C3/C4): key = (score descending, index ascending).
-0.0 equals +0.0; NaN ranks below every non-NaN value (incl. -inf), NaNs tie
among themselves and fall back to the index; +-inf are ordinary values.

Child order (ledger C5, "grouping beams spawned from the same
parent ... preserving the relative order of the parent beams"): survivors are
sorted by old index and child c = r*M + j descends from survivors[r].
"""
from __future__ import annotations

import math
from typing import List, Sequence, Tuple


class SelectError(ValueError):
    pass


def order_key(score: float, index: int):
    s = float(score)
    if math.isnan(s):
        return (1, 0.0, index)
    if s == 0.0:
        s = 0.0  # -0.0 == +0.0
    return (0, -s, index)


def select_survivors(scores: Sequence[float], M: int) -> Tuple[List[int], List[int]]:
    """Return (survivors sorted by index [K], parent map new->old [N])."""
    N = len(scores)
    if N == 0:
        raise SelectError("no active beams")
    if M <= 0 or N % M != 0:
        raise SelectError("N % M != 0")
    K = N // M
    order = sorted(range(N), key=lambda i: order_key(scores[i], i))
    survivors = sorted(order[:K])
    parent = [survivors[c // M] for c in range(N)]
    return survivors, parent


# ---------------------------------------------------------------------------
# Selection variants.  PAPER.md P:182: "Diverse Selection
# ... improve[s] diversity by choosing the top candidate from distinct
# subtrees, while Dynamic Branching ... makes the branching factor itself
# adaptive to verifier scores"; both are "variants of the core beam search
# algorithm".  The paper gives no formula; the readings (DESIGN.md
# ledger C23/C24) follow SPEC S:44 and S:68.

def select_diverse(scores: Sequence[float], B: int) -> Tuple[List[int], List[int]]:
    """Diverse selection (DVTS): the N beams form B subtrees of N/B consecutive
    beams (DFS order, ledger C5: subtree s = beams [s N/B, (s+1) N/B)); the top
    beam of each subtree (key C3/C4) survives and spawns N/B children, which
    form subtree s again ("top beam of each, branch count n/B each").
    Returns (survivors [B], parent map new -> old [N])."""
    N = len(scores)
    if N == 0:
        raise SelectError("no active beams")
    if B <= 0 or N % B != 0:
        raise SelectError("N % B != 0")
    n = N // B
    survivors = [min(range(s * n, (s + 1) * n), key=lambda i: order_key(scores[i], i)) for s in range(B)]
    return survivors, [survivors[c // n] for c in range(N)]


def dynamic_weight(score: float) -> float:
    """A survivor's weight: its score, with NaN / negative / non-finite as 0."""
    s = float(score)
    return s if math.isfinite(s) and s > 0.0 else 0.0


def branch_counts_dynamic(survivor_scores: Sequence[float], N: int) -> List[int]:
    """Largest-remainder apportionment of the N children over the K survivors
    by score-proportional weights, with a floor of one child each:
    quota q_i = (N - K) w_i / sum(w) (float64, the sum in survivor order; all
    weights 0 -> equal weights), c_i = 1 + floor(q_i), and the N - sum(c)
    remaining children go one each to the largest fractional parts q_i -
    floor(q_i), ties to the lower survivor index."""
    K = len(survivor_scores)
    w = [dynamic_weight(s) for s in survivor_scores]
    W = 0.0
    for x in w:
        W += x
    if W == 0.0:
        w, W = [1.0] * K, float(K)
    q = [(N - K) * x / W for x in w]
    c = [1 + math.floor(x) for x in q]
    rest = N - sum(c)
    order = sorted(range(K), key=lambda i: (-(q[i] - math.floor(q[i])), i))
    for i in order[:rest]:
        c[i] += 1
    return c


def select_dynamic(scores: Sequence[float], M: int) -> Tuple[List[int], List[int], List[int]]:
    """Dynamic branching: the K = N/M survivors of beam search (top-K by key,
    sorted by index), each with a score-proportional number of children
    (``branch_counts_dynamic``), children contiguous per survivor in survivor
    order (ledger C5).  Returns (survivors, counts, parent map)."""
    survivors, _ = select_survivors(scores, M)
    counts = branch_counts_dynamic([scores[s] for s in survivors], len(scores))
    parent: List[int] = []
    for s, k in zip(survivors, counts):
        parent += [s] * k
    return survivors, counts, parent


POLICY_TOPK, POLICY_DIVERSE, POLICY_DYNAMIC = 0, 1, 2


def select_policy(scores: Sequence[float], policy: int, param: int) -> List[int]:
    """Parent map (new -> old) of one of the three selection rules."""
    if policy == POLICY_TOPK:
        return select_survivors(scores, param)[1]
    if policy == POLICY_DIVERSE:
        return select_diverse(scores, param)[1]
    if policy == POLICY_DYNAMIC:
        return select_dynamic(scores, param)[2]
    raise SelectError(f"unknown policy {policy}")
