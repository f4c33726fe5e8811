"""Rank model of one request whose beams span G GPUs (oracle; test
infrastructure only).

The paper is single-GPU; "top-K candidates globally"
is kept across ranks by SURVEY.md 8(e) and ledger C19/C20, whose rules this
module writes out plainly:

* global beam id (gid) = index in the request's global DFS-ordered beam array;
  the selection key's index is the gid (C19), so survivors and parent maps are
  those of the single-GPU oracle (``select.select_survivors``).
* each rank r holds cap[r] beams (sum = N); local row order = ascending gid.
  At install rank r holds the contiguous gids [sum(cap[:r]), sum(cap[:r+1]))
  (all beams hold the prompt only, so every cut is byte-balanced).
* placement after a fork (8(e) step 3): walk the children in gid order (=
  survivors in gid order, child c = s*M + j, C5); a child stays on its
  parent's rank while that rank has capacity left; the overflow children, in
  ascending gid, go to the lowest rank with free capacity.
* migration (8(e) step 4): a rank imports the whole lineage (every token) of
  each remote parent one of its children needs, in ascending parent gid, into
  spare rows n_old, n_old + 1, ... (fresh pages, lowest free ids, position
  order); then it forks its rows by an explicit parent map: new row i (the
  i-th of its children in gid order) <- the parent's local row; refcounts
  recounted, pages that drop to 0 released before any allocation, then eager
  copy-on-write of a partially filled last page for every child but the first
  (in new-row order) of the same parent (C6-C8).
* page ids are per rank (each rank has its own allocator, C20).
* f4, cross-GPU deduplication (an extension of 8(e); DESIGN.md ledger C31):
  an imported lineage reuses the longest run of its leading FULL pages that
  one of the destination's pre-fork beams holds with the same tokens (ties to
  the lowest gid): the imported row references that beam's first m pages and
  allocates only the remaining ones.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

from .block_table import BlockTableSim
from .select import select_survivors


def placement(parent_gid: Sequence[int], old_rank: Sequence[int], caps: Sequence[int]) -> List[int]:
    """child gid -> rank."""
    N = len(parent_gid)
    assert sum(caps) == N
    fill = [0] * len(caps)
    child_rank = [-1] * N
    for c in range(N):
        r = old_rank[parent_gid[c]]
        if fill[r] < caps[r]:
            child_rank[c] = r
            fill[r] += 1
    for c in range(N):
        if child_rank[c] < 0:
            r = next(q for q in range(len(caps)) if fill[q] < caps[q])
            child_rank[c] = r
            fill[r] += 1
    return child_rank


@dataclass
class RankForkPlan:
    children: List[int]                     # this rank's new beams (gids, ascending)
    imports: List[int]                      # remote parent gids to import, ascending
    parent_rows: List[int]                  # new row i -> old local row (imports at n_old + k)


def rank_plans(parent_gid: Sequence[int], old_gids: Sequence[Sequence[int]], child_rank: Sequence[int]
               ) -> List[RankForkPlan]:
    G = len(old_gids)
    row_of = [{g: i for i, g in enumerate(gs)} for gs in old_gids]
    plans = []
    for r in range(G):
        children = [c for c in range(len(parent_gid)) if child_rank[c] == r]
        imports = sorted({parent_gid[c] for c in children if parent_gid[c] not in row_of[r]})
        slot = {p: len(old_gids[r]) + k for k, p in enumerate(imports)}
        rows = [row_of[r][parent_gid[c]] if parent_gid[c] in row_of[r] else slot[parent_gid[c]] for c in children]
        plans.append(RankForkPlan(children, imports, rows))
    return plans


class RankSim(BlockTableSim):
    """BlockTableSim plus the two operations of a spanning fork."""

    def import_lineage(self, req: int, row: int, ident: Sequence, share_row: int = -1, m: int = 0) -> None:
        P = self.P
        n = len(ident)
        shared = list(self.tables[req][share_row][:m]) if m else []
        for p in shared:
            self.ref[p] += 1
        pages = [self._alloc() for _ in range(-(-n // P) - m)]
        for p in pages:
            self.ref[p] = 1
        if self.track:
            for i, tok in enumerate(ident):
                if i >= m * P:
                    self.content[pages[i // P - m]][i % P] = tok
        rows, lens = self.tables[req], self.lens[req]
        assert row == len(rows)
        rows.append(shared + pages)
        lens.append(n)

    def fork_map(self, req: int, parent_rows: Sequence[int]) -> None:
        P = self.P
        old_rows, old_lens = self.tables[req], self.lens[req]
        new_rows = [list(old_rows[p]) for p in parent_rows]
        new_lens = [old_lens[p] for p in parent_rows]
        touched = set()
        for row in old_rows:
            for p in row:
                self.ref[p] -= 1
                touched.add(p)
        for row in new_rows:
            for p in row:
                self.ref[p] += 1
        for p in sorted(touched):
            if self.ref[p] == 0:
                self._release(p)
        seen = set()
        for i, par in enumerate(parent_rows):
            rem = new_lens[i] % P
            if par in seen and rem:
                src = new_rows[i][-1]
                newp = self._alloc()
                self._copy_tokens(newp, src, rem)
                new_rows[i][-1] = newp
                self.ref[src] -= 1
                self.ref[newp] = 1
            seen.add(par)
        self.tables[req] = new_rows
        self.lens[req] = new_lens


@dataclass
class SpanFork:
    parent_gid: List[int]
    child_rank: List[int]
    plans: List[RankForkPlan]
    tables: List[List[List[int]]] = field(default_factory=list)   # per rank, after the fork
    lens: List[List[int]] = field(default_factory=list)
    ref: List[List[int]] = field(default_factory=list)
    free: List[List[int]] = field(default_factory=list)


class SpanModel:
    """One request of N beams over G ranks, driven like ``OracleRun`` (append by
    gid activity, fork by gid-indexed scores)."""

    def __init__(self, N: int, caps: Sequence[int], num_pages: int, P: int, prompt_len: int,
                 req: int = 0, track_content: bool = True, dedup: bool = False):
        assert sum(caps) == N
        self.N, self.caps, self.P, self.req = N, list(caps), P, req
        self.G = len(caps)
        self.dedup = dedup
        self.migrated_tokens = 0
        self.deduped_tokens = 0
        self.sims = [RankSim(num_pages, P, track_content) for _ in caps]
        starts = [sum(caps[:r]) for r in range(self.G)]
        self.gids = [list(range(starts[r], starts[r] + caps[r])) for r in range(self.G)]
        for r, sim in enumerate(self.sims):
            ids = [("p", req, i) for i in range(prompt_len)] if track_content else None
            sim.init_request(req, caps[r], prompt_len, ids)

    def rank_of(self) -> List[int]:
        out = [-1] * self.N
        for r, gs in enumerate(self.gids):
            for g in gs:
                out[g] = r
        return out

    def append(self, active_by_gid: Sequence[int], ident_by_gid: Optional[Sequence] = None) -> None:
        for r, sim in enumerate(self.sims):
            act = [int(active_by_gid[g]) for g in self.gids[r]]
            ids = None if ident_by_gid is None else [[ident_by_gid[g] for g in self.gids[r]]]
            sim.append([self.req], [act], ids)

    def lens_by_gid(self) -> List[int]:
        out = [0] * self.N
        for r, sim in enumerate(self.sims):
            for i, g in enumerate(self.gids[r]):
                out[g] = sim.lens[self.req][i]
        return out

    def gather(self, gid: int) -> list:
        r = self.rank_of()[gid]
        return self.sims[r].gather(self.req, self.gids[r].index(gid))

    def fork(self, scores_by_gid: Sequence[float], M: int) -> SpanFork:
        _, parent = select_survivors(list(scores_by_gid), M)
        old_rank = self.rank_of()
        child_rank = placement(parent, old_rank, self.caps)
        plans = rank_plans(parent, self.gids, child_rank)
        # lineages leave their source rank before any rank changes (a parent's
        # rows are read at its pre-fork state)
        lineages = {}
        for pl in plans:
            for p in pl.imports:
                src = old_rank[p]
                sim = self.sims[src]
                row = self.gids[src].index(p)
                lineages[p] = sim.gather(self.req, row) if sim.track else [None] * sim.lens[self.req][row]
        rec = SpanFork(parent, child_rank, plans)
        # f4: the longest run of leading full pages of p that a pre-fork beam
        # of the destination holds with the same tokens (ties: lowest gid)
        old_gids = [list(g) for g in self.gids]
        pre = {g: self.gather(g) for gs in old_gids for g in gs} if self.dedup else {}
        for r, (sim, pl) in enumerate(zip(self.sims, plans)):
            for k, p in enumerate(pl.imports):
                m, share = 0, -1
                if self.dedup:
                    for y in old_gids[r]:
                        lcp = 0
                        for a, b in zip(lineages[p], pre[y]):
                            if a != b:
                                break
                            lcp += 1
                        if lcp // self.P > m:
                            m, share = lcp // self.P, y
                n = len(lineages[p])
                self.migrated_tokens += n - m * self.P
                self.deduped_tokens += m * self.P
                sim.import_lineage(self.req, len(self.gids[r]) + k, lineages[p],
                                   old_gids[r].index(share) if m else -1, m)
            sim.fork_map(self.req, pl.parent_rows)
            self.gids[r] = list(pl.children)
        for sim in self.sims:
            rec.tables.append([list(row) for row in sim.tables[self.req]])
            rec.lens.append(list(sim.lens[self.req]))
            rec.ref.append(list(sim.ref))
            rec.free.append(sim.free_set())
        return rec
