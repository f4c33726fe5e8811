"""GPU edge cases and long-chain parity (round 2): the device KV accounting
against the oracle's, V outside the fp16 range, prompt length 0 on the
tcgen05 path, recovery after a sticky error in a split-tile launch, C4 with 16
requests and C5's full 32 x 256-token chains."""
import math

import numpy as np
import pytest
import torch

from oracle.run import OracleRun, default_num_pages
from synth import workload
from gpu_helpers import run_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, scope="module")
def _built():
    from paper_2509_00195_b200 import build
    build.build()
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"


def _sparse(cfg, beams, layers, every):
    def f(it):
        if it.t % every and not it.forks:
            return []
        return [(r, b, l) for k, r in enumerate(it.reqs) for b in beams if b < cfg.N and it.active[k][b]
                for l in layers]
    return f


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_block_table_stats_every_iteration(name):
    """tts_block_table_stats (the algorithmic bytes of every bench roofline)
    equals BlockTableSim.stats (ledger C22) at every iteration."""
    from paper_2509_00195_b200.runner import BeamStepRunner
    cfg = workload.CONFIGS[name]
    if name == "C2":
        cfg = cfg.with_(n_steps=3)
    pages = default_num_pages(cfg, cfg.R)
    orc = OracleRun(cfg, num_pages=pages, track_content=False)
    tr = orc.run(stats=True, snapshot_refs=False)
    runner = BeamStepRunner(cfg, num_pages=pages, gen_device="cpu")
    n_it = len(tr.unique_tokens)
    accum = torch.zeros(n_it, 2, dtype=torch.int64, device=runner.dev)
    state = {"i": 0}

    def on_iter(it, out, active):
        loc = [runner.local[r] for r in it.reqs]
        runner.ctx.tts_block_table_stats(loc, active, accum[state["i"]])
        state["i"] += 1

    runner.run(on_iter=on_iter)
    got = accum.cpu().numpy()
    assert state["i"] == n_it
    assert got[:, 0].tolist() == tr.unique_tokens
    assert got[:, 1].tolist() == tr.logical_tokens


@pytest.mark.parametrize("d,G", [(128, 6), (64, 2)])
@pytest.mark.parametrize("where", ["prompt", "append"])
def test_v_beyond_fp16_range_is_status_2(d, G, where):
    """V is held in fp16 (DESIGN 4, reading C14'): a finite |v| >= 65520 has no
    fp16 value and must raise the sticky TTS_ERR_UNSUPPORTED (2), never store
    inf.  Both attention paths, at install and at append."""
    from paper_2509_00195_b200.runner import BeamStepRunner
    cfg = workload.Config("vbig", R=1, N=4, M=2, L=2, Hq=2 * G, Hkv=2, d=d, P=16, prompt=20, n_steps=2,
                          step_len=8, seed=77)
    r = BeamStepRunner(cfg, num_pages=64, gen_device="cpu")
    k, v = r.inputs.prompt_kv(0)
    if where == "prompt":
        v = v.clone()
        v[1, 7, 1, 3] = 70000.0
        r.ctx.tts_block_table_init_request(0, cfg.N, cfg.prompt, k, v)
    else:
        r.ctx.tts_block_table_init_request(0, cfg.N, cfg.prompt, k, v)
        q, kn, vn = r.inputs.step(0, [0])
        vn = vn.clone()
        vn[0, 0, 2, 1, 5] = -1.0e5
        out = torch.empty(cfg.L, 1, cfg.N, cfg.Hq, cfg.d, dtype=torch.float32, device=r.dev)
        r.ctx.tts_decode_step([0], None, kn, vn, q, 1.0 / math.sqrt(d), out)
    assert r.ctx.tts_device_status() == 2
    # the pool never holds a non-finite V (beam 0's pages: written before the
    # error, or by the failing kernel itself; later kernels are no-ops)
    snap = r.ctx.tts_block_table_snapshot(0, with_pool_state=False)
    pages = sorted({int(p) for p in snap["tables"][0][: -(-int(snap["lens"][0]) // 16)]})
    vp = r.ctx.v_pool.view(cfg.L, -1, 2 * 16 * d)[:, pages]
    assert len(pages) > 0 and torch.isfinite(vp.float()).all()
    # the 65504 boundary (largest finite fp16, exact in bf16) is accepted
    r2 = BeamStepRunner(cfg, num_pages=64, gen_device="cpu")
    k, v = r2.inputs.prompt_kv(0)
    v = v.clone()
    v[0, 3, 0, 0] = 65280.0  # largest bf16 below 65520
    r2.ctx.tts_block_table_init_request(0, cfg.N, cfg.prompt, k, v)
    assert r2.ctx.tts_device_status() == 0


def test_prompt_zero_on_tcgen05_path():
    """An empty prompt (every beam starts with no context; the first decode
    token attends only to itself) on the tcgen05 path (d = 128, G = 6)."""
    cfg = workload.Config("p0", R=2, N=8, M=2, L=2, Hq=12, Hkv=2, d=128, P=16, prompt=0, n_steps=3,
                          step_len=0, ln_mu=math.log(20), ln_sigma=1.0, ln_cap=50, seed=606)
    run_parity(cfg, _sparse(cfg, range(cfg.N), range(cfg.L), 1))


def test_recovery_after_sticky_error_in_split_launch():
    """A V overflow in the append of a call whose tiles are all split across
    CTAs (stream-K) sets the sticky status; after tts_device_status clears it
    (which also resets the split-tile merge counters) and the request is
    re-installed, the same context gives bit-identical outputs to a clean one
    (CTAs of one launch take the same skip decision)."""
    from paper_2509_00195_b200.runner import BeamStepRunner
    cfg = workload.Config("split", R=1, N=16, M=4, L=2, Hq=12, Hkv=2, d=128, P=16, prompt=256,
                          n_steps=3, step_len=24, seed=4242)

    def collect(runner):
        outs = []
        runner.run(on_iter=lambda it, out, active: outs.append(out.clone()))
        runner.release()
        return outs

    clean = collect(BeamStepRunner(cfg, num_pages=400, gen_device="cpu"))
    r = BeamStepRunner(cfg, num_pages=400, gen_device="cpu")
    step = r.inputs.step

    def poisoned(t, greqs):
        q, k, v = step(t, greqs)
        if t == 5:
            v = v.clone()
            v[1, 0, 3, 0, 0] = 1.0e6
        return q, k, v

    r.inputs.step = poisoned
    r.run(max_iters=12)
    assert r.ctx.tts_device_status() == 2
    r.release()
    assert r.ctx.tts_device_status() == 0
    r.inputs.step = step
    again = collect(r)
    assert len(again) == len(clean)
    for a, b in zip(again, clean):
        assert torch.equal(a, b)


def test_repeated_request_in_one_call_is_rejected_without_side_effects():
    from paper_2509_00195_b200.runner import BeamStepRunner
    from paper_2509_00195_b200.tts import TTSError
    cfg = workload.C2.with_(R=2, L=2, n_steps=2, step_len=8)
    r = BeamStepRunner(cfg, num_pages=200, gen_device="cpu")
    r.install()
    q, k, v = r.inputs.step(0, [0, 1])
    out = torch.empty(cfg.L, 2, cfg.N, cfg.Hq, cfg.d, dtype=torch.float32, device=r.dev)
    before = r.ctx.tts_seq_lens_host(0).copy()
    with pytest.raises(TTSError) as e:
        r.ctx.tts_decode_step([0, 0], None, k, v, q, 1.0, out)
    assert e.value.code == 1
    assert np.array_equal(r.ctx.tts_seq_lens_host(0), before)
    r.ctx.tts_decode_step([0, 1], None, k, v, q, 1.0, out)
    assert (r.ctx.tts_seq_lens_host(0)[: cfg.N] == before[: cfg.N] + 1).all()
    assert r.ctx.tts_device_status() == 0


def test_c4_sixteen_requests():
    """C4 shapes (1.5B heads, N = 256, M = 4, log-normal straggler steps) with
    16 requests batched per call, 2 TTS steps, 2 layers."""
    cfg = workload.C4.with_(R=16, n_steps=2, L=2)
    run_parity(cfg, _sparse(cfg, [0, 77, 255], [0, 1], 251), check_refs=False)


def test_c5_full_chains_n64_slice():
    """C5's full 32 x 256-token chains (8448 tokens per beam, 31 forks of
    M = 8) on an N = 64 slice, one layer: the long split-KV merges."""
    cfg = workload.C5.with_(N=64, L=1)
    res = run_parity(cfg, _sparse(cfg, [0, 33, 63], [0], 1021), check_refs=False)
    assert res["n_forks"] == 31


@pytest.mark.parametrize("name,budgets", [("C2", [16, 40, 160, 10 ** 6]), ("C3", [64, 400, 2000])])
def test_dpas_plan_and_batched_decode(name, budgets):
    """f3: tts_dpas_plan on the device tables equals the oracle's greedy
    schedule, first-fit tries and eviction cost (oracle/dpas.py, pinned to
    SPEC S:150-199 and Appendix A) at every fork; decoding the beams trie by
    trie (one call per trie, as a memory-bounded server would) gives the same
    outputs within 2e-3 of the oracle."""
    from oracle.dpas import eviction_cost, greedy_schedule, pack_tries
    from paper_2509_00195_b200.runner import BeamStepRunner
    cfg = workload.CONFIGS[name].with_(n_steps=3, step_len=64, L=2)
    pages = default_num_pages(cfg, 1)
    orc = OracleRun(cfg, num_pages=pages, track_content=False)
    plans = []

    def on_fork_orc(run, rec):
        cots = [list(row) for row in run.sim.tables[0]]
        g = greedy_schedule(cots)
        for bud in budgets:
            tries = pack_tries(g, cots, bud)
            cost, shared = eviction_cost(tries, cots)
            plans.append((g, tries, cost, shared))

    orc.run(on_fork=on_fork_orc, snapshot_refs=False)
    runner = BeamStepRunner(cfg, num_pages=pages, gen_device="cpu")
    got = []

    def on_fork(it, parents):
        for bud in budgets:
            order, trie_of, nt, cost, shared = runner.ctx.tts_dpas_plan(0, bud)
            tries = [[b for b in order if trie_of[b] == t] for t in range(nt)]
            got.append((order, tries, cost, shared))

    runner.run(on_fork=on_fork)
    assert got == plans and len(got) == (cfg.n_steps - 1) * len(budgets)


def test_dpas_batched_decode_matches_oracle():
    from paper_2509_00195_b200.runner import BeamStepRunner
    cfg = workload.C2.with_(n_steps=3, step_len=40, L=2)
    sample = _sparse(cfg, range(cfg.N), range(cfg.L), 7)
    orc = OracleRun(cfg, num_pages=default_num_pages(cfg, 1), track_content=False)
    tr = orc.run(sample=sample, snapshot_refs=False)
    runner = BeamStepRunner(cfg, num_pages=default_num_pages(cfg, 1), gen_device="cpu")
    runner.dpas_budget = 24  # pages: a few beams per trie
    outs = {}
    seen_tries = []

    def on_iter(it, out, active):
        for (r, b, l) in sample(it):
            outs[(it.t, r, b, l)] = out[l, 0, b].double().cpu().numpy()
        seen_tries.append(runner.last_n_tries)

    runner.run(on_iter=on_iter)
    assert max(seen_tries) > 1
    for key, ref in tr.outputs.items():
        e = float((np.abs(outs[key] - ref).max(-1) / np.abs(ref).max(-1)).max())
        assert e <= 2e-3, (key, e)
