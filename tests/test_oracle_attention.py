"""Pins for oracle.attention (CPU): closed forms, invariants, the fp64 library
SDPA and the split/merge identity (SURVEY.md 8(c) "What pins each part")."""
import math

import numpy as np
import pytest
import torch

from oracle.attention import attention_fp64, merge_states, partial_state
from oracle.run import OracleRun
from synth import workload


def _rand(seed, n, Hq=4, Hkv=2, d=16, qs=1.0):
    rs = np.random.RandomState(seed)
    return rs.randn(Hq, d) * qs, rs.randn(n, Hkv, d), rs.randn(n, Hkv, d)


def test_one_key_returns_v():
    q, K, V = _rand(0, 1)
    o = attention_fp64(q, K, V, 0.25)
    assert np.array_equal(o, np.repeat(V[0], 2, axis=0))


def test_uniform_weights_give_mean():
    q, K, V = _rand(1, 9)
    o = attention_fp64(np.zeros_like(q), K, V, 0.25)          # q = 0
    assert np.allclose(o, np.repeat(V.mean(axis=0), 2, axis=0), atol=1e-14)
    Ks = np.repeat(K[:1], 9, axis=0)                             # identical keys
    o = attention_fp64(q, Ks, V, 0.25)
    assert np.allclose(o, np.repeat(V.mean(axis=0), 2, axis=0), atol=1e-14)


def test_two_keys_sigmoid():
    q, K, V = _rand(2, 2, Hq=2, Hkv=1)
    sc = 0.3
    o = attention_fp64(q, K, V, sc)
    for h in range(2):
        s1, s2 = K[0, 0] @ q[h] * sc, K[1, 0] @ q[h] * sc
        w1 = 1.0 / (1.0 + math.exp(-(s1 - s2)))
        assert np.allclose(o[h], w1 * V[0, 0] + (1 - w1) * V[1, 0], atol=1e-14)


def test_gqa_head_mapping():
    # consecutive q heads share kv head h // G: heads 0,1 see kv 0; 2,3 see kv 1
    q, K, V = _rand(3, 5, Hq=4, Hkv=2)
    q[1] = q[0]
    q[3] = q[2]
    o = attention_fp64(q, K, V, 0.2)
    assert np.array_equal(o[0], o[1]) and np.array_equal(o[2], o[3])
    K2 = K.copy()
    K2[:, 1] *= 2.0  # touching kv head 1 changes only heads 2,3
    o2 = attention_fp64(q, K2, V, 0.2)
    assert np.array_equal(o[:2], o2[:2]) and not np.allclose(o[2:], o2[2:])


def test_permutation_invariance():
    q, K, V = _rand(4, 33)
    perm = np.random.RandomState(0).permutation(33)
    assert np.allclose(attention_fp64(q, K, V, 0.2), attention_fp64(q, K[perm], V[perm], 0.2), atol=1e-13)


@pytest.mark.parametrize("seed,n,Hq,Hkv,d,qs", [(5, 1, 4, 2, 64, 1.0), (6, 77, 12, 2, 128, 1.0),
                                                 (7, 300, 28, 4, 128, 4.0), (8, 16, 7, 7, 32, 1.0)])
def test_library_sdpa(seed, n, Hq, Hkv, d, qs):
    q, K, V = _rand(seed, n, Hq, Hkv, d, qs)
    G = Hq // Hkv
    sc = 1.0 / math.sqrt(d)
    tq = torch.from_numpy(q).view(1, Hq, 1, d)
    tk = torch.from_numpy(K).permute(1, 0, 2).repeat_interleave(G, dim=0).unsqueeze(0)
    tv = torch.from_numpy(V).permute(1, 0, 2).repeat_interleave(G, dim=0).unsqueeze(0)
    ref = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv, scale=sc)[0, :, 0].numpy()
    assert np.abs(attention_fp64(q, K, V, sc) - ref).max() <= 1e-12


@pytest.mark.parametrize("seed", range(6))
def test_split_merge_identity(seed):
    rs = np.random.RandomState(100 + seed)
    n = int(rs.randint(2, 400))
    q, K, V = _rand(seed, n, 14, 2, 64, 4.0 if seed % 2 else 1.0)
    cuts = sorted(set(rs.randint(1, n, size=rs.randint(1, 6)).tolist()))
    parts = np.split(np.arange(n), cuts)
    states = [partial_state(q, K[p], V[p], 0.125) for p in parts]
    m, l, o = merge_states(states)
    full = attention_fp64(q, K, V, 0.125)
    assert np.abs(o - full).max() <= 1e-12
    m1, l1, _ = partial_state(q, K, V, 0.125)
    assert np.allclose(m, m1) and np.allclose(l, l1, rtol=1e-12)


def test_oracle_run_c1_outputs_are_sdpa_of_gathered_pages():
    """End to end on C1: the per-beam (list) attention equals SDPA over K/V
    gathered through the block-table simulator's pages."""
    cfg = workload.C1
    run = OracleRun(cfg)
    tr = run.run(sample=lambda it: [(r, b, 0) for r in it.reqs for b in range(cfg.N) if it.t % 7 == 0])
    assert tr.beam_steps == cfg.N * cfg.n_steps * cfg.step_len
    assert len(tr.forks) == cfg.n_steps - 1
    assert len(tr.outputs) > 0
    for (t, r, b, l), o in tr.outputs.items():
        assert o.shape == (cfg.Hq, cfg.d) and np.isfinite(o).all()
