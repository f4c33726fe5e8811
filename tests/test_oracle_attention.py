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


def _identity_kv(cfg, ident, l):
    """K/V [n, Hkv, d] of a list of token identities, regenerated from synth by
    the identity definitions of synth/rng.py (prompt token i of request r ->
    *_PROMPT keyed (layer, r, i, kv head); the token beam slot b appended at
    iteration t -> keyed (layer, r, t, b, kv head)).  Written here from those
    definitions, not through oracle.run.KVSource."""
    from synth import rng
    kvh = torch.arange(cfg.Hkv).view(1, -1)
    n = len(ident)
    K = torch.empty(n, cfg.Hkv, cfg.d, dtype=torch.float64)
    V = torch.empty_like(K)
    ip = [k for k, tok in enumerate(ident) if tok[0] == "p"]
    idd = [k for k, tok in enumerate(ident) if tok[0] == "d"]
    if ip:
        r = torch.tensor([ident[k][1] for k in ip]).view(-1, 1)
        i = torch.tensor([ident[k][2] for k in ip]).view(-1, 1)
        K[ip] = rng.kv_prompt_values(cfg.seed, "k", l, r, i, kvh, cfg.d).double()
        V[ip] = rng.kv_prompt_values(cfg.seed, "v", l, r, i, kvh, cfg.d).double()
    if idd:
        r, t, b = (torch.tensor([ident[k][j] for k in idd]).view(-1, 1) for j in (1, 2, 3))
        K[idd] = rng.kv_decode_values(cfg.seed, "k", l, r, t, b, kvh, cfg.d).double()
        V[idd] = rng.kv_decode_values(cfg.seed, "v", l, r, t, b, kvh, cfg.d).double()
    return K, V


def _sdpa_default_scale(q, K, V, G):
    """fp64 library SDPA at its DEFAULT scale (1/sqrt(d), ledger C10), GQA expanded."""
    Hq, d = q.shape
    tq = q.view(1, Hq, 1, d)
    tk = K.permute(1, 0, 2).repeat_interleave(G, dim=0).unsqueeze(0)
    tv = V.permute(1, 0, 2).repeat_interleave(G, dim=0).unsqueeze(0)
    return torch.nn.functional.scaled_dot_product_attention(tq, tk, tv)[0, :, 0].numpy()


@pytest.mark.parametrize("cfg", [
    workload.C1,
    # partial prompt page (37 tokens), straggler steps, G = 3, >= 2 forks
    workload.Config("pin-rand", R=2, N=6, M=3, L=2, Hq=6, Hkv=2, d=32, P=16, prompt=37, n_steps=4,
                    step_len=0, ln_mu=math.log(9), ln_sigma=0.8, ln_cap=30, seed=31337, q_scale=4.0),
], ids=["C1", "rand-partial-prompt"])
def test_oracle_beam_output_is_sdpa_over_block_table_gather(cfg):
    """Pins OracleRun.beam_output (ledger C10 scale 1/sqrt(d), C11 the new token
    attends to itself, and which tokens make up a beam's context) against an
    independent definition: the beam's token identities read through the
    block-table simulator's pages (BlockTableSim.gather),
    K/V/q regenerated from those identities, fp64 SDPA at its default scale.
    The query of beam b at iteration t is keyed (layer, r, t, b, q head); the
    token it attends to last is the one it appended at t (PAPER.md P:338,
    GenerateOneToken precedes the step's attention; P:148 paged attention)."""
    from synth import rng
    run = OracleRun(cfg)
    gathered = {}

    def sample(it):
        pts = []
        for k, r in enumerate(it.reqs):
            for b in range(cfg.N):
                if it.active[k][b] and (it.t % 3 == 0 or it.forks):
                    gathered[(it.t, r, b)] = run.sim.gather(r, b)
                    pts += [(r, b, l) for l in range(cfg.L)]
        return pts

    tr = run.run(sample=sample)
    assert len(tr.forks) >= 2 and len(tr.outputs) > 0
    hq = torch.arange(cfg.Hq)
    for (t, r, b, l), o in tr.outputs.items():
        ident = gathered[(t, r, b)]
        assert ident[-1] == ("d", r, t, b)  # the token appended at t is the last one attended
        K, V = _identity_kv(cfg, ident, l)
        q = rng.q_values(cfg.seed, l, r, t, b, hq, cfg.d, cfg.q_scale).double()
        ref = _sdpa_default_scale(q, K, V, cfg.G)
        assert np.abs(o - ref).max() <= 1e-12, (t, r, b, l)
