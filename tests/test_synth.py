"""CPU checks of the shared input generator and workload schedule."""
import math

import numpy as np
import torch

from synth import rng, workload


def test_generator_deterministic_and_shaped():
    a = rng.kv_decode_values(7, "k", 3, 0, torch.arange(5).view(-1, 1), 2, torch.arange(4).view(1, -1), 128)
    b = rng.kv_decode_values(7, "k", 3, 0, torch.arange(5).view(-1, 1), 2, torch.arange(4).view(1, -1), 128)
    assert a.shape == (5, 4, 128) and a.dtype == torch.bfloat16
    assert torch.equal(a, b)
    c = rng.kv_decode_values(7, "v", 3, 0, torch.arange(5).view(-1, 1), 2, torch.arange(4).view(1, -1), 128)
    assert not torch.equal(a, c)


def test_generator_moments():
    x = rng.normal_bf16((1, 2, torch.arange(4096)), 128).float()
    assert abs(x.mean().item()) < 0.01
    assert abs(x.std().item() - 65536 / math.sqrt(3) / 32768) < 0.01
    assert x.abs().max().item() <= 4.0


def test_mix32_known_values():
    # lowbias32 reference values computed with Python ints (exact)
    def ref(x):
        x &= 0xFFFFFFFF
        x ^= x >> 16
        x = (x * 0x7FEB352D) & 0xFFFFFFFF
        x ^= x >> 15
        x = (x * 0x846CA68B) & 0xFFFFFFFF
        x ^= x >> 16
        return x
    xs = [0, 1, 2, 0xFFFFFFFF, 0x12345678, 2509001]
    got = rng.mix32(torch.tensor(xs, dtype=torch.int64)).tolist()
    assert got == [ref(x) for x in xs]


def test_scores_grid():
    s = workload.scores(workload.C4, 3, 2)
    assert s.dtype == torch.float32 and s.shape == (256,)
    assert ((s * 64) == torch.round(s * 64)).all() and (s >= 0).all() and (s < 1).all()


def test_step_lengths_lognormal_shape():
    L = workload.step_lengths(workload.C4)
    assert L.shape == (64, 8, 256) and L.min() >= 1 and L.max() <= 2048
    # heavy tail: max >= 5x mean over 10^4+ draws
    assert L.max() >= 5 * L.mean()
    assert abs(np.median(L) - 200) < 15  # median of LogNormal(ln 200, 1) = 200
    cap1 = workload.step_lengths(workload.C4.with_(ln_cap=1))
    assert (cap1 == 1).all()


def test_schedule_counts():
    cfg = workload.C1
    its = list(workload.schedule(cfg))
    assert len(its) == cfg.n_steps * cfg.step_len
    assert sum(len(i.forks) for i in its) == cfg.n_steps - 1
    cfg = workload.C4.with_(R=3)
    its = list(workload.schedule(cfg))
    lens = workload.step_lengths(cfg)
    total = sum(int(a.sum()) for i in its for a in i.active)
    assert total == int(lens.sum())
    assert sum(len(i.forks) for i in its) == cfg.R * (cfg.n_steps - 1)
