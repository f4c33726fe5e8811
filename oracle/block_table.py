"""Sequential paged block-table simulator (oracle; test infrastructure only).

A page holds P consecutive tokens of one beam for every layer (ledger C9).
Rules (SURVEY.md 8(c) ledger, the readings of a paper that is silent here):

* C7 allocation: the lowest free page id first; within one call every release
  happens before any allocation; allocations are served in (call order of the
  requests, beam/child index) order; a prompt's pages are allocated in
  position order before any copy-on-write page.
* C8 refcount: ref[p] = number of live beam tables containing p (SPEC S:89
  "ref_count equals the number of currently resident paths whose lineage
  includes this node").  A page is free iff ref[p] == 0.
* C6 eager copy-on-write: at install, beams 1..N-1 get a private copy of a
  partially filled last prompt page; at fork, child j = c mod M >= 1 gets a
  private copy of its parent's partially filled last page, child j = 0 keeps
  the original.  Invariant: the page receiving a beam's next token has ref 1.
* C11/C12 append: every active beam appends one token; a beam with
  len % P == 0 first allocates a page.
* Fork ("replicated", P:347 DuplicateThenTruncate with no truncation,
  P:394 siblings grouped): new row c = old row of survivors[c // M].

Page contents are tracked as token identities so that gathering a beam through
its table can be compared with the per-beam explicit list.
"""
from __future__ import annotations

import heapq
from typing import Dict, List, Optional, Sequence

from .select import select_survivors


class OutOfPages(RuntimeError):
    pass


class BlockTableSim:
    def __init__(self, num_pages: int, P: int, track_content: bool = True):
        self.num_pages = num_pages
        self.P = P
        self.free_heap: List[int] = list(range(num_pages))
        heapq.heapify(self.free_heap)
        self.is_free = [True] * num_pages
        self.ref = [0] * num_pages
        self.track = track_content
        self.content: Dict[int, list] = {}
        self.tables: Dict[int, List[List[int]]] = {}
        self.lens: Dict[int, List[int]] = {}

    # -- allocator -----------------------------------------------------------
    def _alloc(self) -> int:
        if not self.free_heap:
            raise OutOfPages("pool exhausted")
        p = heapq.heappop(self.free_heap)
        assert self.is_free[p] and self.ref[p] == 0
        self.is_free[p] = False
        if self.track:
            self.content[p] = [None] * self.P
        return p

    def _release(self, p: int) -> None:
        assert self.ref[p] == 0 and not self.is_free[p]
        self.is_free[p] = True
        heapq.heappush(self.free_heap, p)
        if self.track:
            self.content.pop(p, None)

    def _copy_tokens(self, dst: int, src: int, n: int) -> None:
        if self.track:
            self.content[dst][:n] = self.content[src][:n]

    # -- a1: request install -------------------------------------------------
    def init_request(self, req: int, n_beams: int, prompt_len: int,
                     prompt_ids: Optional[Sequence] = None) -> None:
        assert req not in self.tables
        P = self.P
        npg = -(-prompt_len // P)
        pages = [self._alloc() for _ in range(npg)]
        if self.track:
            for i in range(prompt_len):
                self.content[pages[i // P]][i % P] = prompt_ids[i] if prompt_ids is not None else ("p", req, i)
        rows = [list(pages) for _ in range(n_beams)]
        for p in pages:
            self.ref[p] += n_beams
        rem = prompt_len % P
        if rem:
            last = pages[-1]
            for b in range(1, n_beams):
                newp = self._alloc()
                self._copy_tokens(newp, last, rem)
                rows[b][-1] = newp
                self.ref[last] -= 1
                self.ref[newp] = 1
        self.tables[req] = rows
        self.lens[req] = [prompt_len] * n_beams

    # -- a2: per-token append --------------------------------------------------
    def append(self, reqs: Sequence[int], actives: Sequence[Sequence[int]],
               ids: Optional[Sequence[Sequence]] = None) -> None:
        P = self.P
        for k, r in enumerate(reqs):
            rows, lens = self.tables[r], self.lens[r]
            for b, a in enumerate(actives[k]):
                if not a:
                    continue
                if lens[b] % P == 0:
                    p = self._alloc()
                    rows[b].append(p)
                    self.ref[p] = 1
                page = rows[b][lens[b] // P]
                assert self.ref[page] == 1, "write into a shared page"
                if self.track:
                    self.content[page][lens[b] % P] = ids[k][b] if ids is not None else ("d", r, b, lens[b])
                lens[b] += 1

    # -- a6 + a7: select and fork ---------------------------------------------
    def fork(self, reqs: Sequence[int], scores: Sequence[Sequence[float]], M: int):
        """Returns the parent maps (new -> old) per request."""
        P = self.P
        parents = []
        new_tables, new_lens = {}, {}
        for k, r in enumerate(reqs):
            _, parent = select_survivors(list(scores[k]), M)
            parents.append(parent)
            new_tables[r] = [list(self.tables[r][parent[c]]) for c in range(len(parent))]
            new_lens[r] = [self.lens[r][parent[c]] for c in range(len(parent))]
        # releases first (C7): recount references
        touched = set()
        for r in reqs:
            for row in self.tables[r]:
                for p in row:
                    self.ref[p] -= 1
                    touched.add(p)
            for row in new_tables[r]:
                for p in row:
                    self.ref[p] += 1
        for p in sorted(touched):
            if self.ref[p] == 0:
                self._release(p)
        # then eager CoW allocations in (request, child) order (C6/C7)
        for r in reqs:
            rows, lens = new_tables[r], new_lens[r]
            for c in range(len(rows)):
                j = c % M
                rem = lens[c] % P
                if j >= 1 and rem != 0:
                    src = rows[c][-1]
                    newp = self._alloc()
                    self._copy_tokens(newp, src, rem)
                    rows[c][-1] = newp
                    self.ref[src] -= 1
                    self.ref[newp] = 1
            self.tables[r] = rows
            self.lens[r] = lens
        return parents

    def fork_parents(self, reqs: Sequence[int], parents: Sequence[Sequence[int]]) -> None:
        """Fork by explicit parent maps (selection variants): new
        row c = old row parents[c]; releases before allocations (C7); eager CoW
        of a partially filled last page for every child that is not the first
        child of its parent (children of a parent are contiguous, C5; for
        beam search this is child j = c mod M >= 1, C6)."""
        P = self.P
        new_tables, new_lens = {}, {}
        for k, r in enumerate(reqs):
            par = parents[k]
            new_tables[r] = [list(self.tables[r][par[c]]) for c in range(len(par))]
            new_lens[r] = [self.lens[r][par[c]] for c in range(len(par))]
        touched = set()
        for r in reqs:
            for row in self.tables[r]:
                for p in row:
                    self.ref[p] -= 1
                    touched.add(p)
            for row in new_tables[r]:
                for p in row:
                    self.ref[p] += 1
        for p in sorted(touched):
            if self.ref[p] == 0:
                self._release(p)
        for k, r in enumerate(reqs):
            par = parents[k]
            rows, lens = new_tables[r], new_lens[r]
            for c in range(len(rows)):
                rem = lens[c] % P
                if c > 0 and par[c] == par[c - 1] and rem != 0:
                    src = rows[c][-1]
                    newp = self._alloc()
                    self._copy_tokens(newp, src, rem)
                    rows[c][-1] = newp
                    self.ref[src] -= 1
                    self.ref[newp] = 1
            self.tables[r] = rows
            self.lens[r] = lens

    def release_request(self, req: int) -> None:
        for row in self.tables.pop(req):
            for p in row:
                self.ref[p] -= 1
                if self.ref[p] == 0:
                    self._release(p)
        self.lens.pop(req)

    # -- views -------------------------------------------------------------------
    def free_set(self) -> List[int]:
        return [p for p in range(self.num_pages) if self.is_free[p]]

    def gather(self, req: int, beam: int) -> list:
        """Token identities of a beam read through its table."""
        P = self.P
        n = self.lens[req][beam]
        row = self.tables[req][beam]
        return [self.content[row[i // P]][i % P] for i in range(n)]

    def stats(self, reqs: Sequence[int], actives: Sequence[Sequence[int]]):
        """(unique_tokens, logical_tokens) over active beams (ledger C22):
        unique = sum over distinct pages touched of their valid tokens."""
        P = self.P
        valid = {}
        logical = 0
        for k, r in enumerate(reqs):
            for b, a in enumerate(actives[k]):
                if not a:
                    continue
                n = self.lens[r][b]
                logical += n
                for i, p in enumerate(self.tables[r][b][: -(-n // P)]):
                    valid[p] = max(valid.get(p, 0), min(P, n - i * P))
        return sum(valid.values()), logical
