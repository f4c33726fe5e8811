"""GPU: Speculative Beam Extension, decode side (f1; Alg. 1
P:324-350) through libtts against the oracle (oracle/spec.py): at every fork
the parent map (equal to the run without speculation -- algorithmic
equivalence), the children's source rows and lengths
(DuplicateThenTruncate), tables, refcounts and free set bit-exact; the rows
running at every iteration identical; sampled attention rows of originals
and branches within 2e-3."""
import math

import numpy as np
import pytest
import torch

from oracle.spec import SpecRun
from synth import workload

pytestmark = pytest.mark.gpu
TOL = 2e-3


@pytest.fixture(autouse=True, scope="module")
def _built():
    from paper_2509_00195_b200 import build
    build.build()
    assert torch.cuda.is_available()


def _cfg(seed, d=128, G=6, N=8, M=2, R=1, L=2, prompt=21):
    return workload.Config(f"spec{seed}", R=R, N=N, M=M, L=L, Hq=G * 2, Hkv=2, d=d, P=16, prompt=prompt, n_steps=4,
                           step_len=0, ln_mu=math.log(14), ln_sigma=1.0, ln_cap=60, seed=9100 + seed)


def _parity(cfg, spec=True, every=5):
    from paper_2509_00195_b200.runner import SpecBeamRunner

    def sample(t, r, rows):
        return [(row, l) for row in rows if t % every == 0 for l in range(cfg.L)]

    orc = SpecRun(cfg, spec)
    tr = orc.run(sample=sample)
    run = SpecBeamRunner(cfg, spec=spec, num_pages=orc.num_pages, gen_device="cpu")
    run.ctx.k_pool.fill_(float("nan"))
    run.ctx.v_pool.fill_(float("nan"))
    got, forks = {}, []

    def on_iter(t, reqs, rows_of, out):
        for i, r in enumerate(reqs):
            for row, l in sample(t, r, rows_of[r]):
                got[(t, r, row, l)] = out[l, i, row].double().cpu().numpy()

    def on_fork(t, r, parent, prow, nlen):
        snap = run.ctx.tts_block_table_snapshot(r, with_pool_state=True)
        forks.append({"t": t, "req": r, "parent": parent, "parent_rows": prow, "new_lens": nlen, "snap": snap})

    stats = run.run(on_iter=on_iter, on_fork=on_fork)
    assert run.ctx.tts_device_status() == 0
    assert stats["running"] == tr.running and stats["iterations"] == tr.iterations
    assert len(forks) == len(tr.forks)
    for f, o in zip(forks, tr.forks):
        assert (f["t"], f["req"]) == (o["t"], o["req"])
        assert f["parent"] == o["parent"] and f["parent_rows"] == o["parent_rows"] and f["new_lens"] == o["new_lens"]
        sn = f["snap"]
        assert sn["lens"].tolist() == o["new_lens"]
        for b, row in enumerate(o["tables"]):
            assert sn["tables"][b][: len(row)].tolist() == row, (f["t"], b)
        assert sn["ref"].tolist() == o["ref"] and sn["free"].tolist() == o["free"]
    assert set(got) == set(tr.outputs) and len(got) > 0
    for key, ref in tr.outputs.items():
        e = float((np.abs(got[key] - ref).max(-1) / np.abs(ref).max(-1)).max())
        assert e <= TOL, (key, e)
    return tr, stats


@pytest.mark.parametrize("seed,d,G,N,M,R", [(0, 128, 6, 8, 2, 1), (1, 128, 7, 16, 4, 2), (2, 64, 2, 8, 4, 1),
                                            (3, 128, 4, 16, 2, 1)])
def test_spec_parity(seed, d, G, N, M, R):
    _parity(_cfg(seed, d, G, N, M, R))


def test_spec_equivalence_and_occupancy_on_gpu():
    """Same survivors with speculation on and off; higher slot occupancy and
    no more iterations with it (C4-shaped straggler steps, 1.5B heads)."""
    cfg = workload.C4.with_(R=2, N=16, n_steps=3, L=1, ln_cap=300)
    on_tr, on = _parity(cfg, True, every=97)
    off_tr, off = _parity(cfg, False, every=97)
    assert [f["parent"] for f in on_tr.forks] == [f["parent"] for f in off_tr.forks]
    occ_on = sum(on["running"]) / sum(on["capacity"])
    occ_off = sum(off["running"]) / sum(off["capacity"])
    assert occ_on >= occ_off and on["iterations"] <= off["iterations"]
    print(f"occupancy {occ_off:.3f} -> {occ_on:.3f}; iterations {off['iterations']} -> {on['iterations']}")
