"""GPU tests of a request whose beams span G ranks,
through libtts's own cross-rank step (tts_beam_select_fork_global):

* G contexts on one GPU, one thread per rank over the host transport
  (ThreadGroup, "fake ranks");
* a one-rank NCCL communicator (the NCCL path of the library);
* two processes sharing cuda:0 over a gloo group (GlooTransport).

Every fork is compared with the CPU rank model (oracle/ranks.py: placement,
migration and per-rank allocators written from 8(e) / ledger C19-C20): global
parent map, child -> rank, and per rank the beams' gids, tables, lengths,
refcounts and free set, bit-exact.  Sampled attention rows (by global beam id)
are compared with the single-rank oracle within 2e-3."""
import math
import os
import threading

import numpy as np
import pytest
import torch

from oracle.ranks import SpanModel
from oracle.run import OracleRun
from synth import workload

pytestmark = pytest.mark.gpu

TOL = 2e-3


def _ctx(cfg, caps, pages):
    from paper_2509_00195_b200.runner import tts_config
    from paper_2509_00195_b200.tts import Context
    c = Context(tts_config(cfg, 1, num_pages=pages, max_beams=2 * max(caps)))
    c.k_pool.fill_(float("nan"))
    c.v_pool.fill_(float("nan"))
    return c


def _rows(x, gids, max_beams):
    """Rows `gids` of a [L][1][N][H][d] input, in the call layout
    [L][1][max_beams][H][d] (beam stride = the context's max_beams)."""
    out = torch.zeros(x.shape[0], 1, max_beams, *x.shape[3:], dtype=x.dtype, device=x.device)
    out[:, :, : len(gids)] = x.index_select(2, torch.tensor(gids, device=x.device))
    return out


def _decode(ctx, cfg, it, q, k, v, scale):
    """This rank's decode call: its beams (ascending gid) of iteration it."""
    gids = ctx.tts_span_gids(0)
    mb = ctx.cfg.max_beams
    a = np.zeros((1, mb), dtype=np.uint8)
    a[0, : len(gids)] = it.active[0][gids]
    out = torch.empty(cfg.L, 1, mb, cfg.Hq, cfg.d, dtype=torch.float32, device=q.device)
    ctx.tts_decode_step([0], a, _rows(k, gids, mb), _rows(v, gids, mb), _rows(q, gids, mb), scale, out)
    return gids, out


def _compare_rank(ctx, rec, r, P, gids_model, where):
    snap = ctx.tts_block_table_snapshot(0, with_pool_state=True)
    assert ctx.tts_span_gids(0) == gids_model, f"{where}: gids"
    assert snap["lens"].tolist() == rec.lens[r], f"{where}: lens"
    for b, row in enumerate(rec.tables[r]):
        assert snap["tables"][b][: len(row)].tolist() == row, f"{where}: table row {b}"
    assert np.array_equal(snap["ref"], np.array(rec.ref[r], dtype=np.int32)), f"{where}: refcounts"
    assert snap["free"].tolist() == rec.free[r], f"{where}: free set"


def _span_run(cfg, caps, transports, sample_every=7, pages=None, dedup=False):
    """Drive one spanning request through G contexts (rank r uses transports[r],
    or NCCL when transports is the string "nccl1"); compare with the models."""
    from paper_2509_00195_b200 import build
    build.build()
    from paper_2509_00195_b200.runner import Inputs, pages_per_request

    G = len(caps)
    dev = torch.device("cuda", 0)
    pages = pages or pages_per_request(cfg) + 256
    ctxs = [_ctx(cfg, caps, pages) for _ in range(G)]
    inp = Inputs(cfg, dev, "cpu")
    kp, vp = inp.prompt_kv(0)
    stage = None
    for r, c in enumerate(ctxs):
        c.tts_block_table_init_request(0, caps[r], cfg.prompt, kp, vp)
        if transports == "nccl1":
            from paper_2509_00195_b200.tts import comm_unique_id
            stage = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
            c.tts_comm_init(comm_unique_id(), 1, 0, stage)
        else:
            c.tts_comm_init_host(G, r, transports[r], stage_bytes=256 << 20)
        c.tts_span_init(0, cfg.N, caps, dedup)

    def sample(it):
        if it.t % sample_every:
            return []
        return [(0, g, l) for g in range(0, cfg.N, max(1, cfg.N // 6)) if it.active[0][g] for l in range(cfg.L)]

    orc = OracleRun(cfg, num_pages=pages * G)
    tr = orc.run(sample=sample)
    model = SpanModel(N=cfg.N, caps=caps, num_pages=pages, P=cfg.P, prompt_len=cfg.prompt, dedup=dedup)
    scale = 1.0 / math.sqrt(cfg.d)
    got, n_fork = {}, 0
    for it in workload.schedule(cfg, [0]):
        q, k, v = inp.step(it.t, [0])
        act = it.active[0]
        model.append(act.tolist(), [("d", 0, it.t, g) for g in range(cfg.N)])
        for r, c in enumerate(ctxs):
            gids, out = _decode(c, cfg, it, q, k, v, scale)
            for (_, g, l) in sample(it):
                if g in gids:
                    got[(it.t, 0, g, l)] = out[l, 0, gids.index(g)].double().cpu().numpy()
        for (_, s) in it.forks:
            sc = inp.scores(0, s)
            rec = model.fork(sc.cpu().tolist(), cfg.M)
            orec = tr.forks[n_fork]
            assert rec.parent_gid == orec.parents[0]
            outs = [(torch.empty(cfg.N, dtype=torch.int32, device=dev), torch.empty(cfg.N, dtype=torch.int32, device=dev))
                    for _ in range(G)]
            errs = []

            def work(r):
                try:
                    gids = ctxs[r].tts_span_gids(0)
                    loc = sc[torch.tensor(gids, device=sc.device)].contiguous()
                    ctxs[r].tts_beam_select_fork_global(0, loc, cfg.M, outs[r][0], outs[r][1])
                except Exception as e:  # noqa: BLE001
                    errs.append((r, e))

            th = [threading.Thread(target=work, args=(r,)) for r in range(G)]
            for t_ in th:
                t_.start()
            for t_ in th:
                t_.join()
            assert not errs, errs
            for r in range(G):
                assert outs[r][0].cpu().tolist() == rec.parent_gid, f"fork {n_fork} rank {r}: parent"
                assert outs[r][1].cpu().tolist() == rec.child_rank, f"fork {n_fork} rank {r}: child rank"
                _compare_rank(ctxs[r], rec, r, cfg.P, model.gids[r], f"fork {n_fork} rank {r}")
            n_fork += 1
    for c in ctxs:
        assert c.tts_device_status() == 0
    assert n_fork == len(tr.forks)
    assert model.lens_by_gid() == orc.sim.lens[0]
    assert set(got) == set(tr.outputs)
    for key, ref in tr.outputs.items():
        e = float((np.abs(got[key] - ref).max(-1) / np.abs(ref).max(-1)).max())
        assert e <= TOL, (key, e)
    # migration traffic: what every rank sent (and saved) equals the model's tokens x bytes per token
    tok_bytes = 2 * cfg.L * cfg.Hkv * cfg.d * 2
    sent = [c.tts_span_stats(0) for c in ctxs]
    assert sum(x[0] for x in sent) == model.migrated_tokens * tok_bytes
    assert sum(x[1] for x in sent) == model.deduped_tokens * tok_bytes
    for c in ctxs:
        c.tts_comm_destroy()
    return n_fork


@pytest.mark.parametrize("G,caps", [(2, [8, 8]), (4, [4, 4, 4, 4]), (3, [6, 2, 8])])
def test_thread_ranks_straggler_steps(G, caps):
    from paper_2509_00195_b200.dist import ThreadGroup
    cfg = workload.Config("span-small", R=1, N=sum(caps), M=4, L=2, Hq=28, Hkv=4, d=128, P=16, prompt=37,
                          n_steps=4, step_len=0, ln_mu=math.log(12), ln_sigma=1.0, ln_cap=40, seed=5150 + G)
    grp = ThreadGroup(G)
    assert _span_run(cfg, caps, [grp.transport(r) for r in range(G)]) == 3


@pytest.mark.parametrize("G,caps", [(2, [8, 8]), (4, [4, 4, 4, 4])])
def test_thread_ranks_dedup(G, caps):
    """f4: migrated lineages reuse the leading pages the destination holds
    (page origins); per-rank tables / refcounts / free sets bit-exact against
    the deduplicating rank model, fewer bytes migrated, same outputs."""
    from paper_2509_00195_b200.dist import ThreadGroup
    cfg = workload.Config("span-dedup", R=1, N=sum(caps), M=4, L=2, Hq=28, Hkv=4, d=128, P=16, prompt=37,
                          n_steps=4, step_len=0, ln_mu=math.log(40), ln_sigma=0.7, ln_cap=100, seed=6160 + G)
    grp = ThreadGroup(G)
    assert _span_run(cfg, caps, [grp.transport(r) for r in range(G)], dedup=True) == 3


def test_thread_ranks_c5_shape():
    """C5's head shape and branching (M = 8) on 8 ranks, N = 64 of 512."""
    from paper_2509_00195_b200.dist import ThreadGroup
    cfg = workload.C5.with_(N=64, L=1, n_steps=3, step_len=48, prompt=64)
    grp = ThreadGroup(8)
    _span_run(cfg, [8] * 8, [grp.transport(r) for r in range(8)], sample_every=13)


def test_nccl_one_rank_communicator():
    """The NCCL path of tts_beam_select_fork_global (all-gather over a
    one-rank communicator) equals the single-rank oracle."""
    cfg = workload.Config("span-nccl1", R=1, N=16, M=4, L=2, Hq=12, Hkv=2, d=128, P=16, prompt=20, n_steps=4,
                          step_len=0, ln_mu=math.log(10), ln_sigma=1.0, ln_cap=30, seed=777)
    _span_run(cfg, [16], "nccl1")


def _gloo_worker(rank, world, port, queue):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2509_00195_b200 import build
        build.build()
        from paper_2509_00195_b200.dist import GlooTransport
        from paper_2509_00195_b200.runner import Inputs
        cfg = workload.Config("span-gloo", R=1, N=8, M=2, L=1, Hq=14, Hkv=2, d=128, P=16, prompt=21, n_steps=3,
                              step_len=0, ln_mu=math.log(9), ln_sigma=1.0, ln_cap=25, seed=31)
        caps = [4, 4]
        dev = torch.device("cuda", 0)
        ctx = _ctx(cfg, caps, 400)
        inp = Inputs(cfg, dev, "cpu")
        kp, vp = inp.prompt_kv(0)
        ctx.tts_block_table_init_request(0, caps[rank], cfg.prompt, kp, vp)
        ctx.tts_comm_init_host(world, rank, GlooTransport(), stage_bytes=64 << 20)
        ctx.tts_span_init(0, cfg.N, caps, True)
        scale = 1.0 / math.sqrt(cfg.d)
        snaps = []
        for it in workload.schedule(cfg, [0]):
            q, k, v = inp.step(it.t, [0])
            gids, _ = _decode(ctx, cfg, it, q, k, v, scale)
            for (_, s) in it.forks:
                sc = inp.scores(0, s)
                loc = sc[torch.tensor(gids, device=dev)].contiguous()
                par = torch.empty(cfg.N, dtype=torch.int32, device=dev)
                cr = torch.empty(cfg.N, dtype=torch.int32, device=dev)
                ctx.tts_beam_select_fork_global(0, loc, cfg.M, par, cr)
                snap = ctx.tts_block_table_snapshot(0, with_pool_state=True)
                snaps.append({"parent": par.cpu().tolist(), "child_rank": cr.cpu().tolist(),
                              "gids": ctx.tts_span_gids(0), "lens": snap["lens"].tolist(),
                              "tables": [snap["tables"][b][: -(-int(ln) // cfg.P)].tolist()
                                         for b, ln in enumerate(snap["lens"])],
                              "ref": snap["ref"].tolist(), "free": snap["free"].tolist()})
        assert ctx.tts_device_status() == 0
        queue.put((rank, snaps, cfg, caps))
    finally:
        dist.destroy_process_group()


def test_gloo_two_processes_share_cuda0():
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict()
    for _ in range(2):
        r, snaps, cfg, caps = q.get(timeout=600)
        res[r] = snaps
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    model = SpanModel(N=cfg.N, caps=caps, num_pages=400, P=cfg.P, prompt_len=cfg.prompt, dedup=True)
    k = 0
    for it in workload.schedule(cfg, [0]):
        model.append(it.active[0].tolist(), [("d", 0, it.t, g) for g in range(cfg.N)])
        for (_, s) in it.forks:
            rec = model.fork(workload.scores(cfg, 0, s).tolist(), cfg.M)
            for r in range(2):
                sn = res[r][k]
                assert sn["parent"] == rec.parent_gid and sn["child_rank"] == rec.child_rank
                assert sn["gids"] == model.gids[r] and sn["lens"] == rec.lens[r]
                assert sn["tables"] == rec.tables[r]
                assert sn["ref"] == rec.ref[r] and sn["free"] == rec.free[r]
            k += 1
    assert k == len(res[0]) == 2
