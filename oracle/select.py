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
