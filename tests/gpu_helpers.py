"""Shared helpers for the GPU parity tests: run the same seeded workload through
the oracle (CPU) and through libtts (C-ABI on the GPU) and compare."""
from __future__ import annotations

from typing import Callable, Dict, List, Optional, Tuple

import numpy as np

from oracle.run import OracleRun, default_num_pages
from synth import workload

TOL = 2e-3  # north_star: max relative error, read row-normwise (SURVEY ledger C13)


def rownorm_err(got: np.ndarray, ref: np.ndarray) -> float:
    """max over rows of max_k |got - ref| / max_k |ref| (rows = last-but-one axis)."""
    num = np.abs(got - ref).max(axis=-1)
    den = np.abs(ref).max(axis=-1)
    return float((num / den).max())


def compare_state(snap: dict, tables: List[List[int]], lens: List[int], P: int,
                  ref: Optional[np.ndarray], free: Optional[np.ndarray], where: str) -> None:
    N = len(tables)
    assert snap["n_beams"] == N, where
    assert list(snap["lens"]) == list(lens), f"{where}: lens"
    for b in range(N):
        npg = -(-lens[b] // P)
        got = snap["tables"][b][:npg].tolist()
        assert got == list(tables[b]), f"{where}: table row {b}: {got} vs {tables[b]}"
    if ref is not None:
        assert np.array_equal(snap["ref"], ref.astype(np.int32)), f"{where}: refcounts"
    if free is not None:
        assert np.array_equal(snap["free"], free), f"{where}: free set"


def run_parity(cfg: workload.Config, sample: Callable, num_pages: Optional[int] = None,
               scores_fn: Optional[Callable] = None, max_iters: Optional[int] = None,
               check_refs: bool = True, fused: bool = True, policy=None) -> Dict[str, float]:
    from paper_2509_00195_b200.runner import BeamStepRunner

    num_pages = num_pages or default_num_pages(cfg, cfg.R)
    orc = OracleRun(cfg, num_pages=num_pages, track_content=cfg.R * cfg.N <= 64)
    tr = orc.run(sample=sample, snapshot_refs=check_refs, scores_fn=scores_fn, max_iters=max_iters, policy=policy)

    runner = BeamStepRunner(cfg, num_pages=num_pages, fused=fused)
    ctx = runner.ctx
    # poison the pools: slots that are never written must never reach an output
    ctx.k_pool.fill_(float("nan"))
    ctx.v_pool.fill_(float("nan"))
    outs: Dict[Tuple[int, int, int, int], np.ndarray] = {}
    snaps = []

    def on_iter(it, out, active):
        for (r, b, l) in sample(it):
            outs[(it.t, r, b, l)] = out[l, it.reqs.index(r), b].double().cpu().numpy()

    def on_fork(it, parents):
        rec = {"t": it.t, "parents": parents, "snap": {}}
        for r in parents:
            rec["snap"][r] = ctx.tts_block_table_snapshot(runner.local[r], with_pool_state=check_refs)
        snaps.append(rec)

    steps = runner.run(on_iter=on_iter, on_fork=on_fork, max_iters=max_iters, scores_fn=scores_fn, policy=policy)
    assert ctx.tts_device_status() == 0
    assert steps == tr.beam_steps

    # integer state: bit-exact at every fork
    assert len(snaps) == len(tr.forks)
    for rec, orec in zip(snaps, tr.forks):
        assert rec["t"] == orec.t
        for r, par in rec["parents"].items():
            assert list(par) == orec.parents[r], f"t={orec.t} r={r}: parent map"
            compare_state(rec["snap"][r], orec.tables[r], orec.lens[r], cfg.P,
                          orec.ref, orec.free, f"fork t={orec.t} r={r}")
    # end state
    for r in runner.req_ids:
        snap = ctx.tts_block_table_snapshot(runner.local[r], with_pool_state=True)
        ofree = np.array(orc.sim.free_set(), dtype=np.int64)
        compare_state(snap, orc.sim.tables[r], orc.sim.lens[r], cfg.P,
                      np.array(orc.sim.ref), ofree, f"end r={r}")
        assert list(ctx.tts_seq_lens_host(runner.local[r])[: cfg.N]) == orc.sim.lens[r]
    # attention: row-normwise relative error per sampled (t, r, b, l)
    assert set(outs) == set(tr.outputs)
    worst = 0.0
    for key, ref in tr.outputs.items():
        e = rownorm_err(outs[key], ref)
        worst = max(worst, e)
        assert e <= TOL, f"{key}: row-normwise error {e:.3e} > {TOL}"
    return {"worst_err": worst, "n_outputs": len(outs), "n_forks": len(snaps)}
