"""Counter-based generator for synthetic q / k / v / scores.

Every value is a pure function of its identity key (seed, stream, layer,
request, iteration, beam, head, dim).  The hash is Wellons' "lowbias32"
32-bit mixer evaluated on int64 torch tensors holding values in [0, 2^32):
only +, *, ^, >>, & on int64, so CPU and CUDA give bit-identical results.

Normal-ish values: the sum of four independent uniform 16-bit integers
(Irwin-Hall, n=4) centred and divided by 2^15; the result (an integer over a
power of two, |x| <= 4) is exact in fp32 and is then rounded to bf16 with
round-to-nearest-even by ``Tensor.to(torch.bfloat16)`` on either device.
Standard deviation = 65536 / sqrt(3) / 32768 ~= 1.155.

SURVEY.md 2e N9 / 8(d) "Concrete synthetic inputs".
"""
from __future__ import annotations

import torch

M32 = 0xFFFFFFFF

# stream ids (part of the key)
STREAM_Q = 1
STREAM_K = 2
STREAM_V = 3
STREAM_K_PROMPT = 4
STREAM_V_PROMPT = 5
STREAM_SCORE = 6
STREAM_STEPLEN = 7
STREAM_TRUNC = 8


def _mul32(x: torch.Tensor, c: int) -> torch.Tensor:
    """(x * c) mod 2^32 without int64 overflow (x < 2^32, c < 2^32)."""
    lo = c & 0xFFFF
    hi = c >> 16
    return ((x * lo) + (((x * hi) & 0xFFFF) << 16)) & M32


def mix32(x: torch.Tensor) -> torch.Tensor:
    """lowbias32: x ^= x>>16; x *= 0x7feb352d; x ^= x>>15; x *= 0x846ca68b; x ^= x>>16."""
    x = x & M32
    x = x ^ (x >> 16)
    x = _mul32(x, 0x7FEB352D)
    x = x ^ (x >> 15)
    x = _mul32(x, 0x846CA68B)
    x = x ^ (x >> 16)
    return x


def _as_key(v, device) -> torch.Tensor:
    if isinstance(v, torch.Tensor):
        return v.to(device=device, dtype=torch.int64) & M32
    return torch.tensor(int(v) & M32, dtype=torch.int64, device=device)


def hash_key(fields, device="cpu") -> torch.Tensor:
    """Chain-hash a sequence of (broadcastable) integer fields into 32-bit keys."""
    h = mix32(torch.tensor(0x9E3779B9, dtype=torch.int64, device=device))
    for f in fields:
        h = mix32(h ^ _as_key(f, device))
    return h


def normal_bf16(fields, dim: int, device="cpu") -> torch.Tensor:
    """bf16 values ~ N(0, 1.155^2), shape = broadcast(fields) + (dim,)."""
    h = hash_key(fields, device).unsqueeze(-1)
    d = torch.arange(dim, dtype=torch.int64, device=device)
    e0 = mix32(h ^ mix32(2 * d + 0x51ED27))
    e1 = mix32(h ^ mix32(2 * d + 0x51ED28))
    s = (e0 & 0xFFFF) + (e0 >> 16) + (e1 & 0xFFFF) + (e1 >> 16)  # [0, 262140]
    x = (s - 131070).to(torch.float32) / 32768.0  # exact in fp32
    return x.to(torch.bfloat16)


def uniform_u32(fields, device="cpu") -> torch.Tensor:
    return hash_key(fields, device)


# ---------------------------------------------------------------------------
# Named tensors of the workload.  Index conventions (all int tensors or ints):
#   layer l, request r (global id), iteration t (global decode iteration
#   counter of the run), beam b (slot index at generation time), head h.
# ---------------------------------------------------------------------------

def q_values(seed, layer, req, t, beam, qhead, d, q_scale=1.0, device="cpu"):
    x = normal_bf16((seed, STREAM_Q, layer, req, t, beam, qhead), d, device)
    if q_scale != 1.0:
        x = (x.float() * q_scale).to(torch.bfloat16)  # power-of-two scale: exact
    return x


def kv_decode_values(seed, which, layer, req, t, beam, kvhead, d, device="cpu"):
    s = STREAM_K if which == "k" else STREAM_V
    return normal_bf16((seed, s, layer, req, t, beam, kvhead), d, device)


def kv_prompt_values(seed, which, layer, req, pos, kvhead, d, device="cpu"):
    s = STREAM_K_PROMPT if which == "k" else STREAM_V_PROMPT
    return normal_bf16((seed, s, layer, req, pos, kvhead), d, device)


def score_values(seed, req, step, beam, device="cpu") -> torch.Tensor:
    """PRM scores: U[0,1) on a 1/64 grid (tie-heavy). fp32, exact."""
    u = uniform_u32((seed, STREAM_SCORE, req, step, beam), device)
    return ((u >> 26).to(torch.float32) / 64.0)


def score_values_fine(seed, req, step, beam, device="cpu") -> torch.Tensor:
    """Unquantised variant: U[0,1) with 24 random bits (exact in fp32)."""
    u = uniform_u32((seed, STREAM_SCORE, req, step, beam), device)
    return ((u >> 8).to(torch.float32) / float(1 << 24))


def truncation_fraction(seed, req, step, child, mean: float, sigma: float) -> float:
    """Speculative-token truncation fraction f ~ Normal(mean, sigma) clamped to
    [0, 1] for child `child` of the fork after TTS step `step` (PAPER.md P:311
    "drawn from a normal distribution with mean R"; SPEC S:67 sigma 0.1): a
    random input of DuplicateThenTruncate, drawn here once (float64, Box-Muller
    on two counter-based uniforms) and handed to both the oracle and libtts."""
    import math
    u = [(int(uniform_u32((seed, STREAM_TRUNC, req, step, child, k))) + 0.5) / 4294967296.0 for k in (1, 2)]
    z = math.sqrt(-2.0 * math.log(u[0])) * math.cos(2.0 * math.pi * u[1])
    return min(1.0, max(0.0, mean + sigma * z))
