"""Workload configurations (BASELINE.json ``configs``) and the iteration schedule.

Nothing here is the method's arithmetic: these are the shapes of the paper's
workloads (SURVEY.md 8, table "Shapes used throughout"), the synthetic step
lengths (fixed 256-token steps, or LogNormal(ln 200, 1.0) ceil
clamp [1, 2048] for the straggler-heavy C4), and the order in
which a driver calls append / attention / select-fork:

* all R requests start together on their prompt;
* at global iteration t a request in step s (started at t0) has beam b active
  iff t - t0 < steplen[r][s][b] (Alg. 1 lines 7-14 with B_spec = {},
  SURVEY C12);
* a request whose longest beam finished at iteration t forks after t
  ("Top-scoring paths are then replicated"), except after its last step
  (fixed number of steps).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import Iterator, List, Optional, Tuple

import numpy as np
import torch

from . import rng


@dataclass(frozen=True)
class Config:
    name: str
    R: int            # requests
    N: int            # live beams per request
    M: int            # branching factor (children per survivor); K = N / M
    L: int            # layers
    Hq: int           # query heads
    Hkv: int          # kv heads
    d: int            # head dim
    P: int            # page size (tokens)
    prompt: int       # prompt tokens
    n_steps: int      # TTS steps
    step_len: int = 0             # fixed step length (0 -> log-normal)
    ln_mu: float = math.log(200.0)
    ln_sigma: float = 1.0
    ln_cap: int = 2048
    seed: int = 2509001
    q_scale: float = 1.0
    fine_scores: bool = False
    num_pages: int = 0            # 0 -> derived

    @property
    def G(self) -> int:
        return self.Hq // self.Hkv

    @property
    def K(self) -> int:
        return self.N // self.M

    @property
    def kv_bytes_per_token_layer(self) -> int:
        return 4 * self.Hkv * self.d  # bf16 K and V

    def with_(self, **kw) -> "Config":
        return replace(self, **kw)


# BASELINE.json configs[0..4] (seeds 2509001 + index, 8(d))
C1 = Config("C1-tiny", R=1, N=4, M=2, L=1, Hq=4, Hkv=2, d=64, P=16, prompt=32,
            n_steps=3, step_len=16, seed=2509001)
C2 = Config("C2-qwen2.5-math-1.5b", R=1, N=16, M=4, L=28, Hq=12, Hkv=2, d=128, P=16,
            prompt=256, n_steps=8, step_len=256, seed=2509002)
C3 = Config("C3-qwen2.5-math-7b", R=1, N=64, M=4, L=28, Hq=28, Hkv=4, d=128, P=16,
            prompt=256, n_steps=16, step_len=256, seed=2509003)
C4 = Config("C4-batch64-1.5b-straggler", R=64, N=256, M=4, L=28, Hq=12, Hkv=2, d=128, P=16,
            prompt=256, n_steps=8, step_len=0, seed=2509004)
C5 = Config("C5-span-7b-n512", R=1, N=512, M=8, L=28, Hq=28, Hkv=4, d=128, P=16,
            prompt=256, n_steps=32, step_len=256, seed=2509005)

CONFIGS = {"C1": C1, "C2": C2, "C3": C3, "C4": C4, "C5": C5}


def step_lengths(cfg: Config) -> np.ndarray:
    """int64 [R][n_steps][N] tokens per (request, step, beam)."""
    R, S, N = cfg.R, cfg.n_steps, cfg.N
    if cfg.step_len > 0:
        return np.full((R, S, N), cfg.step_len, dtype=np.int64)
    r = torch.arange(R).view(R, 1, 1)
    s = torch.arange(S).view(1, S, 1)
    b = torch.arange(N).view(1, 1, N)
    u1 = rng.uniform_u32((cfg.seed, rng.STREAM_STEPLEN, r, s, b, 1)).numpy().astype(np.float64)
    u2 = rng.uniform_u32((cfg.seed, rng.STREAM_STEPLEN, r, s, b, 2)).numpy().astype(np.float64)
    u1 = (u1 + 0.5) / 4294967296.0
    u2 = (u2 + 0.5) / 4294967296.0
    z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)
    x = np.exp(cfg.ln_mu + cfg.ln_sigma * z)
    return np.clip(np.ceil(x), 1, cfg.ln_cap).astype(np.int64)


def scores(cfg: Config, req: int, step: int, device="cpu") -> torch.Tensor:
    b = torch.arange(cfg.N, device=device)
    f = rng.score_values_fine if cfg.fine_scores else rng.score_values
    return f(cfg.seed, req, step, b, device=device)


@dataclass
class Iteration:
    t: int
    reqs: List[int]                       # requests with >= 1 active beam, ascending
    active: List[np.ndarray]              # per listed request: uint8 [N]
    forks: List[Tuple[int, int]] = field(default_factory=list)  # (req, step) forking after t
    ends: List[int] = field(default_factory=list)               # requests finished after t


def schedule(cfg: Config, req_ids: Optional[List[int]] = None) -> Iterator[Iteration]:
    """Yield the decode iterations of a whole run for the given requests."""
    lens = step_lengths(cfg)
    req_ids = list(range(cfg.R)) if req_ids is None else list(req_ids)
    step = {r: 0 for r in req_ids}
    t0 = {r: 0 for r in req_ids}
    live = list(req_ids)
    t = 0
    while live:
        it = Iteration(t=t, reqs=[], active=[])
        for r in live:
            sl = lens[r, step[r]]
            act = ((t - t0[r]) < sl).astype(np.uint8)
            it.reqs.append(r)
            it.active.append(act)
            if t - t0[r] + 1 == int(sl.max()):
                if step[r] + 1 < cfg.n_steps:
                    it.forks.append((r, step[r]))
                    step[r] += 1
                    t0[r] = t + 1
                else:
                    it.ends.append(r)
        live = [r for r in live if r not in it.ends]
        yield it
        t += 1


def total_tokens_per_beam_max(cfg: Config) -> int:
    lens = step_lengths(cfg)
    return cfg.prompt + int(lens.max(axis=2).sum(axis=1).max())


def max_pages_per_beam(cfg: Config) -> int:
    return -(-total_tokens_per_beam_max(cfg) // cfg.P)
