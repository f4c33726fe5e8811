"""Whole-configuration oracle driver (test infrastructure only).

Follows the generation/verification loop of PAPER.md 3.1 with the
per-token inner loop of Alg. 1 lines 7-14 (B_spec = {}), driven by the
schedule in ``synth.workload`` (which beams are active at each iteration and
which requests end a step).  Two independent representations are kept:

1. ``lists``   -- per beam, the explicit list of token identities; a fork
                  deep-copies the parent's list ("replicated").
2. ``sim``     -- the sequential block-table simulator (``block_table``).

Attention is computed from (1) only: each beam's K/V are regenerated from its
own identity list (a materialised, unshared copy).
At every fork the two representations are cross-checked (item 7).

Token identity: prompt token i of request r -> K/V from stream *_PROMPT keyed
(layer, r, i, kvhead); the token appended by beam slot b at global iteration t
-> stream K/V keyed (layer, r, t, b, kvhead); the query of beam b at
iteration t -> stream Q keyed (layer, r, t, b, qhead).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch

from synth import rng, workload
from .attention import attention_fp64
from .block_table import BlockTableSim
from .select import select_policy, select_survivors


def default_num_pages(cfg: workload.Config, n_req: int) -> int:
    if cfg.num_pages:
        return cfg.num_pages
    per_beam = workload.max_pages_per_beam(cfg)
    return n_req * cfg.N * per_beam + 64


class KVSource:
    """Regenerates K/V for token identities (the materialised per-beam copy)."""

    def __init__(self, cfg: workload.Config):
        self.cfg = cfg
        self._prompt: Dict[Tuple[int, int, str], torch.Tensor] = {}

    def prompt(self, r: int, l: int, which: str) -> torch.Tensor:
        key = (r, l, which)
        if key not in self._prompt:
            c = self.cfg
            pos = torch.arange(c.prompt).view(-1, 1)
            kvh = torch.arange(c.Hkv).view(1, -1)
            self._prompt[key] = rng.kv_prompt_values(c.seed, which, l, r, pos, kvh, c.d)
        return self._prompt[key]

    def decode(self, r: int, l: int, which: str, ident: np.ndarray) -> torch.Tensor:
        c = self.cfg
        t = torch.from_numpy(np.ascontiguousarray(ident[:, 0])).view(-1, 1)
        b = torch.from_numpy(np.ascontiguousarray(ident[:, 1])).view(-1, 1)
        kvh = torch.arange(c.Hkv).view(1, -1)
        return rng.kv_decode_values(c.seed, which, l, r, t, b, kvh, c.d)

    def beam_kv(self, r: int, l: int, ident: np.ndarray, prompt_len: int):
        Kp = self.prompt(r, l, "k")[:prompt_len]
        Vp = self.prompt(r, l, "v")[:prompt_len]
        if len(ident):
            K = torch.cat([Kp, self.decode(r, l, "k", ident)])
            V = torch.cat([Vp, self.decode(r, l, "v", ident)])
        else:
            K, V = Kp, Vp
        return K.double().numpy(), V.double().numpy()


def q_for(cfg: workload.Config, r: int, t: int, b: int, l: int) -> np.ndarray:
    h = torch.arange(cfg.Hq)
    return rng.q_values(cfg.seed, l, r, t, b, h, cfg.d, cfg.q_scale).double().numpy()


@dataclass
class ForkRecord:
    t: int
    reqs: List[int]
    parents: Dict[int, List[int]]
    tables: Dict[int, List[List[int]]]
    lens: Dict[int, List[int]]
    ref: Optional[np.ndarray] = None
    free: Optional[np.ndarray] = None


@dataclass
class Trace:
    forks: List[ForkRecord] = field(default_factory=list)
    outputs: Dict[Tuple[int, int, int, int], np.ndarray] = field(default_factory=dict)  # (t,r,b,l)
    beam_steps: int = 0
    unique_tokens: List[int] = field(default_factory=list)
    logical_tokens: List[int] = field(default_factory=list)


class OracleRun:
    def __init__(self, cfg: workload.Config, req_ids: Optional[Sequence[int]] = None,
                 num_pages: Optional[int] = None, track_content: bool = True):
        self.cfg = cfg
        self.req_ids = list(range(cfg.R)) if req_ids is None else list(req_ids)
        self.num_pages = num_pages or default_num_pages(cfg, len(self.req_ids))
        self.sim = BlockTableSim(self.num_pages, cfg.P, track_content)
        self.kv = KVSource(cfg)
        self.lists: Dict[int, List[np.ndarray]] = {}
        self.step: Dict[int, int] = {}
        self.track = track_content

    def install(self) -> None:
        c = self.cfg
        for r in self.req_ids:
            ids = [("p", r, i) for i in range(c.prompt)] if self.track else None
            self.sim.init_request(r, c.N, c.prompt, ids)
            self.lists[r] = [np.zeros((0, 2), dtype=np.int64) for _ in range(c.N)]
            self.step[r] = 0

    def beam_output(self, r: int, b: int, t: int, l: int) -> np.ndarray:
        c = self.cfg
        K, V = self.kv.beam_kv(r, l, self.lists[r][b], c.prompt)
        return attention_fp64(q_for(c, r, t, b, l), K, V, 1.0 / math.sqrt(c.d))

    def cross_check(self, r: int) -> None:
        """table gather == explicit per-beam list."""
        c = self.cfg
        for b in range(c.N):
            got = self.sim.gather(r, b)
            want = [("p", r, i) for i in range(c.prompt)] + [("d", r, int(t), int(bb)) for t, bb in self.lists[r][b]]
            assert got == want, f"table/list mismatch r={r} b={b}"

    def run(self, sample: Optional[Callable[[workload.Iteration], List[Tuple[int, int, int]]]] = None,
            snapshot_refs: bool = True, stats: bool = False, max_iters: Optional[int] = None,
            scores_fn: Optional[Callable[[int, int], Sequence[float]]] = None,
            on_fork: Optional[Callable[["OracleRun", ForkRecord], None]] = None,
            policy: Optional[Tuple[int, int]] = None) -> Trace:
        """policy: (select.POLICY_*, param) for the selection variants (f2); default
        beam search with the configuration's M."""
        c = self.cfg
        tr = Trace()
        self.install()
        for it in workload.schedule(c, self.req_ids):
            if max_iters is not None and it.t >= max_iters:
                break
            ids = None
            if self.track:
                ids = [[("d", r, it.t, b) for b in range(c.N)] for r in it.reqs]
            self.sim.append(it.reqs, [a.tolist() for a in it.active], ids)
            for k, r in enumerate(it.reqs):
                act = it.active[k]
                idx = np.nonzero(act)[0]
                for b in idx:
                    self.lists[r][b] = np.concatenate([self.lists[r][b], [[it.t, b]]])
                tr.beam_steps += int(act.sum())
            if stats:
                u, lg = self.sim.stats(it.reqs, [a.tolist() for a in it.active])
                tr.unique_tokens.append(u)
                tr.logical_tokens.append(lg)
            if sample is not None:
                for (r, b, l) in sample(it):
                    tr.outputs[(it.t, r, b, l)] = self.beam_output(r, b, it.t, l)
            if it.forks:
                reqs = [r for r, _ in it.forks]
                scs = []
                for r, s in it.forks:
                    sc = scores_fn(r, s) if scores_fn else workload.scores(c, r, s).tolist()
                    scs.append(list(sc))
                if policy is None:
                    parents = self.sim.fork(reqs, scs, c.M)
                else:
                    parents = [select_policy(sc, policy[0], policy[1]) for sc in scs]
                    self.sim.fork_parents(reqs, parents)
                rec = ForkRecord(t=it.t, reqs=reqs, parents={}, tables={}, lens={})
                for k, r in enumerate(reqs):
                    parent = parents[k]
                    if policy is None:
                        assert parent == select_survivors(scs[k], c.M)[1]
                    self.lists[r] = [self.lists[r][parent[cc]].copy() for cc in range(c.N)]
                    rec.parents[r] = parent
                    rec.tables[r] = [list(row) for row in self.sim.tables[r]]
                    rec.lens[r] = list(self.sim.lens[r])
                    if self.track:
                        self.cross_check(r)
                if snapshot_refs:
                    rec.ref = np.array(self.sim.ref, dtype=np.int64)
                    rec.free = np.array(self.sim.free_set(), dtype=np.int64)
                tr.forks.append(rec)
                if on_fork is not None:
                    on_fork(self, rec)
        return tr
