"""Driver of the beam-step hot path through the C-ABI (the call sequence a
serving loop makes): install every request on its prompt, then per decode
iteration append + prefix-shared attention for all layers, and at each step
end select + fork (PAPER.md 3.1 two-stage loop; Alg. 1 lines 7-19).

Inputs are the seeded synthetic tensors of ``synth`` generated directly on the
device (input generation is not part of the method and is excluded from any
timed region by the callers).  Nothing here computes the method: every step
runs in libtts's kernels.
"""
from __future__ import annotations

import math
from typing import Callable, Dict, List, Optional, Sequence

import numpy as np
import torch

from synth import rng, workload
from .tts import Context, TTSConfig


def pages_per_request(cfg: workload.Config) -> int:
    """Upper bound on the live pages of one request.  Fixed-length steps: the
    prompt (+ CoW copies of a partial last prompt page), at most K = N/M
    distinct survivors' segments for every finished step (later forks only
    drop lineages), and N private segments for the current step (+1 page each
    for a CoW'd partial page).  Variable steps: every beam's whole chain."""
    P = cfg.P
    if cfg.step_len > 0:
        seg = -(-cfg.step_len // P) + 1
        return -(-cfg.prompt // P) + cfg.N + (cfg.n_steps - 1) * cfg.K * seg + cfg.N * seg
    # variable steps (C4): every beam's pages of the current step, plus K
    # survivors per finished step at 1.5x the step's mean length (survivors are
    # chosen by score, not length); a pool that runs out raises the sticky
    # TTS_ERR_OUT_OF_PAGES, it never corrupts state
    lens = workload.step_lengths(cfg)                      # [R][S][N]
    pages = -(-lens // P)
    cur = (pages.sum(axis=2) + cfg.N).max(axis=1)          # [R]
    past = (1.5 * pages.mean(axis=2) + 1).sum(axis=1) * cfg.K
    return int(-(-cfg.prompt // P) + cfg.N + (cur + past).max())


def tts_config(cfg: workload.Config, n_req: int, num_pages: Optional[int] = None,
               max_pages_per_beam: Optional[int] = None, max_beams: Optional[int] = None) -> TTSConfig:
    mp = max_pages_per_beam or workload.max_pages_per_beam(cfg)
    if num_pages is None:
        num_pages = cfg.num_pages or (n_req * pages_per_request(cfg) + 64)
    return TTSConfig(num_layers=cfg.L, num_q_heads=cfg.Hq, num_kv_heads=cfg.Hkv, head_dim=cfg.d,
                     page_size=cfg.P, max_requests=n_req, max_beams=max_beams or cfg.N, max_pages_per_beam=mp,
                     num_pages=int(num_pages))


class Inputs:
    """Identity-keyed synthetic q / k / v / scores on the device.  gen_device:
    where the hash runs ("cpu": generated on the host, bit-identical, then
    copied -- keeps the device's launch stream to libtts's own kernels)."""

    def __init__(self, cfg: workload.Config, device, gen_device=None):
        self.cfg = cfg
        self.out_dev = device
        self.dev = device if gen_device is None else torch.device(gen_device)

    def _idx(self, n, shape_pos, ndim):
        s = [1] * ndim
        s[shape_pos] = n
        return torch.arange(n, device=self.dev).view(*s)

    def prompt_kv(self, req: int):
        c = self.cfg
        l = self._idx(c.L, 0, 3)
        pos = self._idx(c.prompt, 1, 3)
        h = self._idx(c.Hkv, 2, 3)
        k = rng.kv_prompt_values(c.seed, "k", l, req, pos, h, c.d, device=self.dev)
        v = rng.kv_prompt_values(c.seed, "v", l, req, pos, h, c.d, device=self.dev)
        return k.contiguous().to(self.out_dev), v.contiguous().to(self.out_dev)

    def step(self, t: int, greqs: Sequence[int], rows: Optional[int] = None):
        """q [L][n][rows][Hq][d], k/v [L][n][rows][Hkv][d] for global requests greqs
        (rows = beam slots, default N; row b keyed as beam b)."""
        c = self.cfg
        l = self._idx(c.L, 0, 4)
        r = torch.tensor(list(greqs), device=self.dev).view(1, -1, 1, 1)
        b = self._idx(rows or c.N, 2, 4)
        hq = self._idx(c.Hq, 3, 4)
        hk = self._idx(c.Hkv, 3, 4)
        q = rng.q_values(c.seed, l, r, t, b, hq, c.d, c.q_scale, device=self.dev)
        k = rng.kv_decode_values(c.seed, "k", l, r, t, b, hk, c.d, device=self.dev)
        v = rng.kv_decode_values(c.seed, "v", l, r, t, b, hk, c.d, device=self.dev)
        return (q.contiguous().to(self.out_dev), k.contiguous().to(self.out_dev),
                v.contiguous().to(self.out_dev))

    def scores(self, greq: int, step: int):
        return workload.scores(self.cfg, greq, step, device=self.dev).to(self.out_dev)


class BeamStepRunner:
    def __init__(self, cfg: workload.Config, req_ids: Optional[Sequence[int]] = None, device: int = 0,
                 num_pages: Optional[int] = None, fused: bool = True, gen_device=None):
        self.cfg = cfg
        self.fused = fused
        self.req_ids = list(range(cfg.R)) if req_ids is None else list(req_ids)
        self.local = {r: i for i, r in enumerate(self.req_ids)}
        self.tcfg = tts_config(cfg, len(self.req_ids), num_pages)
        self.ctx = Context(self.tcfg, device)
        self.dev = self.ctx.device
        self.inputs = Inputs(cfg, self.dev, gen_device)
        self.scale = 1.0 / math.sqrt(cfg.d)
        # f3: decode in DPAS tries under a KV budget (pages; None = one call for all beams)
        self.dpas_budget: Optional[int] = None
        self.last_n_tries = 1
        self._tries = None

    def _plan_tries(self):
        """DPAS tries of request 0 (the schedule is made once per TTS step,
        PAPER.md Appendix A.1 assumption 2)."""
        order, trie_of, nt, _, _ = self.ctx.tts_dpas_plan(0, self.dpas_budget)
        self._tries = [[b for b in order if trie_of[b] == t] for t in range(nt)]

    def install(self):
        for r in self.req_ids:
            k, v = self.inputs.prompt_kv(r)
            self.ctx.tts_block_table_init_request(self.local[r], self.cfg.N, self.cfg.prompt, k, v)

    def release(self):
        for r in self.req_ids:
            self.ctx.tts_block_table_release_request(self.local[r])

    def run(self, on_iter: Optional[Callable] = None, on_fork: Optional[Callable] = None,
            max_iters: Optional[int] = None, scores_fn: Optional[Callable] = None, policy=None) -> int:
        """Whole run; returns beam-steps.  on_iter(it, out, q) after attention;
        on_fork(it, parents {greq: np.ndarray}) after each fork.  policy:
        (tts.SELECT_*, param) for the selection variants (default beam search, M)."""
        c = self.cfg
        self.install()
        beam_steps = 0
        for it in workload.schedule(c, self.req_ids):
            if max_iters is not None and it.t >= max_iters:
                break
            n = len(it.reqs)
            loc = [self.local[r] for r in it.reqs]
            active = np.stack(it.active).astype(np.uint8)
            q, k, v = self.inputs.step(it.t, it.reqs)
            out = torch.empty(c.L, n, c.N, c.Hq, c.d, dtype=torch.float32, device=self.dev)
            if self.dpas_budget is not None:
                assert len(self.req_ids) == 1 and self.fused, "DPAS batches: one request"
                if self._tries is None:
                    self._plan_tries()
                self.last_n_tries = 0
                for trie in self._tries:
                    a = np.zeros_like(active)
                    a[0, trie] = active[0, trie]
                    if a.any():
                        self.ctx.tts_decode_step(loc, a, k, v, q, self.scale, out)
                        self.last_n_tries += 1
            elif self.fused:
                self.ctx.tts_decode_step(loc, active, k, v, q, self.scale, out)
            else:
                self.ctx.tts_block_table_append(loc, active, k, v)
                self.ctx.tts_prefix_attn_decode(0, c.L, loc, active, q, self.scale, out)
            beam_steps += int(active.sum())
            if on_iter is not None:
                on_iter(it, out, active)
            if it.forks:
                greqs = [r for r, _ in it.forks]
                if scores_fn is not None:
                    sc = torch.stack([torch.as_tensor(scores_fn(r, s), dtype=torch.float32)
                                      for r, s in it.forks]).to(self.dev)
                else:
                    sc = torch.stack([self.inputs.scores(r, s) for r, s in it.forks])
                parent = torch.empty(len(greqs), c.N, dtype=torch.int32, device=self.dev)
                if policy is None:
                    self.ctx.tts_beam_select_fork([self.local[r] for r in greqs], sc.contiguous(), c.M, parent)
                else:
                    self.ctx.tts_beam_select_fork_policy([self.local[r] for r in greqs], sc.contiguous(), policy[0],
                                                         policy[1], parent)
                self._tries = None  # a new schedule for the next step
                if on_fork is not None:
                    on_fork(it, {r: parent[i].cpu().numpy() for i, r in enumerate(greqs)})
        return beam_steps


class SpecBeamRunner:
    """The serving loop of Speculative Beam Extension (Alg. 1, decode
    side; include/tts.h f1) over libtts: per iteration one decode call over
    every request's originals still in their step plus its speculative
    branches; tts_spec_select / tts_spec_branch fill the slots finished beams
    free (from the second step on: the selection needs a previous score); at
    a request's step end, selection over the N original scores
    (tts_beam_select_global), tts_spec_plan and tts_beam_fork_map_trunc.  The
    bookkeeping here is the loop's (remaining tokens per beam, branch token
    counts); every decision is libtts's.  spec=False runs the same loop
    without speculation (the baseline of the same workload)."""

    def __init__(self, cfg: workload.Config, spec: bool = True, R_mean: float = 0.85, R_sigma: float = 0.1,
                 device: int = 0, num_pages: Optional[int] = None, gen_device=None, lengths=None, scores_fn=None):
        self.cfg, self.spec = cfg, spec
        self.R_mean, self.R_sigma = R_mean, R_sigma
        self.maxB = 2 * cfg.N
        pages = num_pages or (cfg.R * 2 * cfg.N * workload.max_pages_per_beam(cfg) + 64)
        self.tcfg = tts_config(cfg, cfg.R, num_pages=pages, max_beams=self.maxB)
        self.ctx = Context(self.tcfg, device)
        self.dev = self.ctx.device
        self.inputs = Inputs(cfg, self.dev, gen_device)
        self.scale = 1.0 / math.sqrt(cfg.d)
        self.lengths = workload.step_lengths(cfg) if lengths is None else np.asarray(lengths)
        self.scores_fn = scores_fn

    def run(self, on_iter: Optional[Callable] = None, on_fork: Optional[Callable] = None) -> dict:
        """on_iter(t, reqs, rows {r: [rows running]}, out) after each decode call;
        on_fork(t, r, parent, parent_rows, new_lens) after each fork.  Returns
        {iterations, running[], capacity[], beam_steps, spec_tokens}."""
        from . import tts as T
        c = self.cfg
        L = self.lengths
        st = {}
        for r in range(c.R):
            k, v = self.inputs.prompt_kv(r)
            self.ctx.tts_block_table_init_request(r, c.N, c.prompt, k, v)
            st[r] = {"s": 0, "rem": [int(x) for x in L[r, 0]], "last": None, "k": [0] * c.N, "br": []}
        stats = {"iterations": 0, "running": [], "capacity": [], "beam_steps": 0, "spec_tokens": 0}
        parent_d = torch.empty(c.N, dtype=torch.int32, device=self.dev)
        t = 0
        while st:
            reqs = sorted(st)
            act = np.zeros((len(reqs), self.maxB), dtype=np.uint8)
            rows_of = {}
            for i, r in enumerate(reqs):
                S = st[r]
                rows = [b for b in range(c.N) if S["rem"][b] > 0] + [c.N + j for j in range(len(S["br"]))]
                act[i, rows] = 1
                rows_of[r] = rows
            q, k, v = self.inputs.step(t, reqs, self.maxB)
            out = torch.empty(c.L, len(reqs), self.maxB, c.Hq, c.d, dtype=torch.float32, device=self.dev)
            self.ctx.tts_decode_step(reqs, act, k, v, q, self.scale, out)
            stats["running"].append(int(act.sum()))
            stats["capacity"].append(c.N * len(reqs))
            for r in reqs:
                S = st[r]
                for b in range(c.N):
                    if S["rem"][b] > 0:
                        S["rem"][b] -= 1
                        stats["beam_steps"] += 1
                S["br"] = [(src, n + 1) for src, n in S["br"]]
                stats["spec_tokens"] += len(S["br"])
            if on_iter is not None:
                on_iter(t, reqs, rows_of, out)
            for r in reqs:
                S = st[r]
                if all(x == 0 for x in S["rem"]):
                    s = S["s"]
                    if s + 1 >= c.n_steps:
                        self.ctx.tts_block_table_release_request(r)
                        del st[r]
                        continue
                    sc = (torch.as_tensor(list(self.scores_fn(r, s)), dtype=torch.float32, device=self.dev)
                          if self.scores_fn else self.inputs.scores(r, s))
                    self.ctx.tts_beam_select_global(sc.contiguous(), c.M, parent_d)
                    parent = parent_d.cpu().tolist()
                    lens = list(self.ctx.tts_seq_lens_host(r)[: c.N])
                    frac = [rng.truncation_fraction(c.seed, r, s, ch, self.R_mean, self.R_sigma) for ch in range(c.N)]
                    nxt = [int(x) for x in L[r, s + 1]]
                    prow, nlen, head = T.spec_plan(parent, c.M, S["br"], lens, frac, nxt)
                    self.ctx.tts_beam_fork_map_trunc(r, prow, nlen)
                    if on_fork is not None:
                        on_fork(t, r, parent, prow, nlen)
                    scl = sc.cpu().tolist()
                    S.update(s=s + 1, rem=[nxt[ch] - head[ch] for ch in range(c.N)],
                             last=[scl[parent[ch]] for ch in range(c.N)], k=[0] * c.N, br=[])
                elif self.spec and S["last"] is not None:
                    free = c.N - sum(1 for x in S["rem"] if x > 0) - len(S["br"])
                    cand = [b for b in range(c.N) if S["rem"][b] == 0]
                    if cand and free > 0:
                        add = T.spec_select(cand, [S["last"][b] for b in cand], [S["k"][b] for b in cand], free, c.M)
                        src = []
                        for b, n in zip(cand, add):  # branch rows in ascending source beam order
                            src += [b] * n
                            S["k"][b] += n
                        if src:
                            self.ctx.tts_spec_branch(r, src)
                            S["br"] += [(b, 0) for b in src]
            t += 1
        stats["iterations"] = t
        return stats
