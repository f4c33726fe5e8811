"""Speculative Beam Extension, decode side (oracle; test infrastructure only).

PAPER.md 4.1, Alg. 1 `SpecBeamExtend`: inside the generation loop
(lines 7-14) beams that finished their thinking step are "speculative
candidates" (SelectSpec, line 12) whose speculative branches run in the slots
the finished beams freed; verification and selection (lines 15-17) see only
the non-speculative step ("algorithmic equivalence"); then
DuplicateThenTruncate (line 18): "only its duplicates have speculative tokens
truncated, while the original remains intact", the truncation length "drawn
from a normal distribution with mean R".  SelectSpec bins the
previous step's score into B bins, M_i = B - j + 1.

The readings (DESIGN.md ledger C25-C29), with SPEC S:240-257:

* bin_score: equal-width bins over [0, 1], C_1 the highest; a score on a
  boundary belongs to the higher bin: j = ceil((1 - s) B) clamped to [1, B]
  (float64; s clamped to [0, 1], NaN -> 0).  M = B - j + 1.  B = the search's
  branching factor M.
* select_spec: candidates = finished beams whose branch count k < M_b;
  sorted by (M_b descending, beam ascending); free slots given greedily,
  each beam at most M_b - k more.  No speculation in the first TTS step
  (no previous score).
* slots: N rows run at a time: originals still in their step + branches.
* a branch is a fork of the finished beam (its table row copied, the
  partially filled last page copied, C6) into a spare row N, N+1, ... (the
  branches granted after one iteration in ascending source beam order, rows
  reset every step); it generates one token per iteration until the step
  ends.
* DuplicateThenTruncate: survivor s's children j = 0..M-1 (child c = r M + j,
  C5): child j < k_s continues from branch j of s with h tokens of it kept --
  all of them for j = 0 (the original's continuation), floor(f n) for j >= 1
  with f ~ Normal(R, sigma) clamped to [0, 1] (drawn by synth, an input);
  children j >= k_s duplicate s (h = 0).  The kept head start is capped at the
  child's next step length; the child then still has L - h tokens to generate.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from .block_table import BlockTableSim
from .select import select_survivors


def bin_score(score: float, B: int) -> Tuple[int, int]:
    """(bin j in 1..B, speculative potential M = B - j + 1)."""
    s = float(score)
    if math.isnan(s):
        s = 0.0
    s = min(1.0, max(0.0, s))
    j = math.ceil((1.0 - s) * B)
    j = min(B, max(1, j))
    return j, B - j + 1


def select_spec(candidates: Sequence[Tuple[int, int, int]], free_slots: int) -> List[Tuple[int, int]]:
    """candidates (beam, M_b, k_b already running) -> [(beam, new branches)]."""
    out = []
    free = free_slots
    for beam, m, k in sorted(candidates, key=lambda x: (-x[1], x[0])):
        if free <= 0:
            break
        n = min(m - k, free)
        if n > 0:
            out.append((beam, n))
            free -= n
    return out


def spec_plan(parent: Sequence[int], M: int, branches: Sequence[Tuple[int, int]], lens: Sequence[int],
              frac: Sequence[float], next_len: Optional[Sequence[int]] = None):
    """DuplicateThenTruncate.  parent: the selection's parent map [N] (child c
    -> surviving beam); branches: per spare row N + i, (source beam, tokens
    generated); lens: the N beams' lengths at the step end; frac: f per child
    (used for j >= 1).  Returns (parent_rows [N]: child -> old row, new_lens [N],
    head [N]: kept speculative tokens)."""
    N = len(parent)
    rows_of: Dict[int, List[int]] = {}
    for i, (src, _) in enumerate(branches):
        rows_of.setdefault(src, []).append(N + i)
    parent_rows, new_lens, head = [], [], []
    for c in range(N):
        s, j = parent[c], c % M
        br = rows_of.get(s, [])
        if j < len(br):
            row = br[j]
            n = branches[row - N][1]
            h = n if j == 0 else math.floor(frac[c] * n)
            if next_len is not None:
                h = min(h, int(next_len[c]))
            parent_rows.append(row)
            new_lens.append(lens[s] + h)
            head.append(h)
        else:
            parent_rows.append(s)
            new_lens.append(lens[s])
            head.append(0)
    return parent_rows, new_lens, head


class SpecSim(BlockTableSim):
    """BlockTableSim plus the two table operations of speculation."""

    def branch(self, req: int, src_rows: Sequence[int]) -> List[int]:
        """New rows (appended) forked from src_rows, in order; a partially filled
        last page is copied into a fresh page for the branch (C6, C7)."""
        P = self.P
        rows, lens = self.tables[req], self.lens[req]
        new = []
        for src in src_rows:
            row = list(rows[src])
            n = lens[src]
            for p in row:
                self.ref[p] += 1
            if n % P:
                old = row[-1]
                newp = self._alloc()
                self._copy_tokens(newp, old, n % P)
                row[-1] = newp
                self.ref[old] -= 1
                self.ref[newp] = 1
            rows.append(row)
            lens.append(n)
            new.append(len(rows) - 1)
        return new

    def fork_trunc(self, req: int, parent_rows: Sequence[int], new_lens: Sequence[int]) -> None:
        """Fork by an explicit map with truncation: new row i = the first
        ceil(new_lens[i] / P) pages of old row parent_rows[i]; releases first
        (C7), then eager CoW of a partially filled last page for every child
        but the first of its parent row (C6).  The first child's partial last
        page keeps the page; its slots past the new length are cleared."""
        P = self.P
        old_rows, old_lens = self.tables[req], self.lens[req]
        new_rows = []
        for pr, n in zip(parent_rows, new_lens):
            assert n <= old_lens[pr]
            new_rows.append(list(old_rows[pr][: -(-n // P)]))
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
        for i, pr in enumerate(parent_rows):
            n = new_lens[i]
            rem = n % P
            if pr in seen and rem:
                src = new_rows[i][-1]
                newp = self._alloc()
                self._copy_tokens(newp, src, rem)
                new_rows[i][-1] = newp
                self.ref[src] -= 1
                self.ref[newp] = 1
            elif rem and self.track:
                page = new_rows[i][-1]
                for k in range(rem, P):
                    self.content[page][k] = None
            seen.add(pr)
        self.tables[req] = new_rows
        self.lens[req] = list(new_lens)


@dataclass
class SpecTrace:
    forks: List[dict] = field(default_factory=list)          # per fork: t, req, parent, parent_rows, new_lens, tables, ref, free
    outputs: Dict[Tuple[int, int, int, int], np.ndarray] = field(default_factory=dict)  # (t, r, row, l)
    running: List[int] = field(default_factory=list)          # rows generating at each iteration (all requests)
    capacity: List[int] = field(default_factory=list)         # N x live requests at each iteration
    iterations: int = 0
    beam_steps: int = 0                                       # non-speculative tokens generated
    spec_tokens: int = 0


class SpecRun:
    """Whole-configuration oracle with speculation on or off (same inputs).
    Per request, step s of beam b lasts L[r][s][b] tokens (synth's step
    lengths), minus the head start its speculative branch left it."""

    def __init__(self, cfg, spec: bool, R_mean: float = 0.85, R_sigma: float = 0.1, num_pages: int = 0,
                 track_content: bool = True, lengths: Optional[np.ndarray] = None, scores_fn=None):
        from synth import workload
        from .run import KVSource
        self.cfg, self.spec = cfg, spec
        self.R_mean, self.R_sigma = R_mean, R_sigma
        self.num_pages = num_pages or (cfg.R * 2 * cfg.N * workload.max_pages_per_beam(cfg) + 64)
        self.sim = SpecSim(self.num_pages, cfg.P, track_content)
        self.kv = KVSource(cfg)
        self.track = track_content
        self.lengths = lengths          # [R][S][N] step lengths (default: synth's)
        self.scores_fn = scores_fn      # (r, s) -> N scores (default: synth's)

    def _output(self, r: int, row: int, t: int, l: int) -> np.ndarray:
        """fp64 attention of row `row` over its own token list (read through its
        table), K/V regenerated from the token identities."""
        from synth import rng
        from .attention import attention_fp64
        import torch
        c = self.cfg
        ident = self.sim.gather(r, row)
        K = np.empty((len(ident), c.Hkv, c.d))
        V = np.empty_like(K)
        kvh = torch.arange(c.Hkv).view(1, -1)
        ip = [i for i, tok in enumerate(ident) if tok[0] == "p"]
        idd = [i for i, tok in enumerate(ident) if tok[0] != "p"]
        if ip:
            K[ip] = self.kv.prompt(r, l, "k")[[ident[i][2] for i in ip]].double().numpy()
            V[ip] = self.kv.prompt(r, l, "v")[[ident[i][2] for i in ip]].double().numpy()
        if idd:
            tt = torch.tensor([ident[i][2] for i in idd]).view(-1, 1)
            bb = torch.tensor([ident[i][3] for i in idd]).view(-1, 1)
            K[idd] = rng.kv_decode_values(c.seed, "k", l, r, tt, bb, kvh, c.d).double().numpy()
            V[idd] = rng.kv_decode_values(c.seed, "v", l, r, tt, bb, kvh, c.d).double().numpy()
        q = rng.q_values(c.seed, l, r, t, row, torch.arange(c.Hq), c.d, c.q_scale).double().numpy()
        return attention_fp64(q, K, V, 1.0 / math.sqrt(c.d))

    def run(self, sample=None) -> SpecTrace:
        """sample(t, r, rows_running) -> [(row, layer)] outputs to record."""
        from synth import rng, workload
        c = self.cfg
        L = workload.step_lengths(c) if self.lengths is None else np.asarray(self.lengths)  # [R][S][N]
        tr = SpecTrace()
        st = {}
        for r in range(c.R):
            ids = [("p", r, i) for i in range(c.prompt)] if self.track else None
            self.sim.init_request(r, c.N, c.prompt, ids)
            st[r] = {"s": 0, "rem": [int(x) for x in L[r, 0]], "last": None, "k": [0] * c.N, "br": []}
        t = 0
        while st:
            running = 0
            for r in sorted(st):
                S = st[r]
                rows = [b for b in range(c.N) if S["rem"][b] > 0] + [c.N + i for i in range(len(S["br"]))]
                act = [0] * (c.N + len(S["br"]))
                for row in rows:
                    act[row] = 1
                ids = [("d", r, t, row) for row in range(len(act))] if self.track else None
                self.sim.append([r], [act], [ids] if ids else None)
                running += len(rows)
                for b in range(c.N):
                    if S["rem"][b] > 0:
                        S["rem"][b] -= 1
                        tr.beam_steps += 1
                for i in range(len(S["br"])):
                    src, n = S["br"][i]
                    S["br"][i] = (src, n + 1)
                    tr.spec_tokens += 1
                if sample is not None:
                    for row, l in sample(t, r, rows):
                        tr.outputs[(t, r, row, l)] = self._output(r, row, t, l)
            tr.running.append(running)
            tr.capacity.append(c.N * len(st))
            for r in sorted(st):
                S = st[r]
                if all(x == 0 for x in S["rem"]):
                    s = S["s"]
                    if s + 1 >= c.n_steps:
                        self.sim.release_request(r)
                        del st[r]
                        continue
                    sc = list(self.scores_fn(r, s)) if self.scores_fn else workload.scores(c, r, s).tolist()
                    _, parent = select_survivors(sc, c.M)
                    lens = self.sim.lens[r][: c.N]
                    frac = [rng.truncation_fraction(c.seed, r, s, ch, self.R_mean, self.R_sigma) for ch in range(c.N)]
                    nxt = [int(x) for x in L[r, s + 1]]
                    prow, nlen, head = spec_plan(parent, c.M, S["br"], lens, frac, nxt)
                    self.sim.fork_trunc(r, prow, nlen)
                    tr.forks.append({"t": t, "req": r, "parent": parent, "parent_rows": prow, "new_lens": nlen,
                                     "head": head, "tables": [list(x) for x in self.sim.tables[r]],
                                     "ref": list(self.sim.ref), "free": self.sim.free_set()})
                    S["s"] = s + 1
                    S["rem"] = [nxt[ch] - head[ch] for ch in range(c.N)]
                    S["last"] = [sc[parent[ch]] for ch in range(c.N)]
                    S["k"] = [0] * c.N
                    S["br"] = []
                elif self.spec and S["last"] is not None:
                    free = c.N - sum(1 for x in S["rem"] if x > 0) - len(S["br"])
                    cand = []
                    for b in range(c.N):
                        if S["rem"][b] == 0:
                            _, m = bin_score(S["last"][b], c.M)
                            if S["k"][b] < m:
                                cand.append((b, m, S["k"][b]))
                    # new branch rows in ascending source beam order (ledger C27)
                    for b, n in sorted(select_spec(cand, free)):
                        self.sim.branch(r, [b] * n)
                        S["br"] += [(b, 0)] * n
                        S["k"][b] += n
            t += 1
        tr.iterations = t
        return tr
