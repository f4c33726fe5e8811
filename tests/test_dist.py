"""Multi-rank host logic of the beam-sharded fork on CPU:
the pure placement / migration plan, and the torch.distributed driver run with
gloo at world size 2 over a mock context (token-identity rows instead of K/V
pages), checked against a single-rank selection and fork."""
import os
import random

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.select import select_survivors
from paper_2509_00195_b200.dist import migration_plan, select_fork_global, shard_requests, transfers


def test_shard_requests_partition():
    for G in (1, 2, 4, 8):
        parts = [shard_requests(64, G, r) for r in range(G)]
        assert sorted(sum(parts, [])) == list(range(64))
        assert max(map(len, parts)) - min(map(len, parts)) <= 1


@pytest.mark.parametrize("seed", range(20))
def test_migration_plan_properties(seed):
    rnd = random.Random(seed)
    G = rnd.choice([2, 4, 8])
    n = rnd.choice([2, 4, 8])
    M = rnd.choice([m for m in (2, 4, 8) if (G * n) % m == 0])
    N = G * n
    scores = [rnd.randint(0, 7) / 8 for _ in range(N)]
    _, parent = select_survivors(scores, M)
    plans = migration_plan(parent, G)
    for r, pl in enumerate(plans):
        assert len(pl.local_parent) == n
        imported = dict((slot, p) for p, slot in pl.imports)
        for i, lp in enumerate(pl.local_parent):
            c = r * n + i
            if lp < n:                       # parent already on this rank
                assert r * n + lp == parent[c]
            else:                            # parent's lineage imported into a spare row
                assert imported[lp] == parent[c] and parent[c] // n != r
        # children of one survivor are consecutive gids (ledger C5)
        assert pl.local_parent == sorted(pl.local_parent) or any(lp >= n for lp in pl.local_parent)
    # every import is matched by exactly one export
    exp = sorted((p, s, d) for s, pl in enumerate(plans) for p, d in pl.exports)
    imp = sorted((p, p // n, d) for d, pl in enumerate(plans) for p, _ in pl.imports)
    assert exp == imp == transfers(plans, G)


class MockCtx:
    """libtts surface over token-identity rows (one request)."""

    def __init__(self, rows):
        self.rows = [list(r) for r in rows]

    def tts_seq_lens_host(self, req):
        return np.array([len(r) for r in self.rows], dtype=np.int32)

    def tts_beam_select_global(self, scores_all, width_m, parent_out):
        _, parent = select_survivors(scores_all.tolist(), width_m)
        parent_out.copy_(torch.tensor(parent, dtype=torch.int32))

    def lineage_buffer(self, length):
        return torch.empty(length, dtype=torch.int64)

    def tts_lineage_export(self, req, beam, buf):
        buf.copy_(torch.tensor(self.rows[beam], dtype=torch.int64))

    def tts_lineage_import(self, req, slot, length, buf):
        while len(self.rows) <= slot:
            self.rows.append([])
        assert not self.rows[slot]
        self.rows[slot] = buf[:length].tolist()

    def tts_beam_fork_map(self, req, local_parent):
        self.rows = [list(self.rows[p]) for p in local_parent]

    def sync(self):
        pass


def _worker(rank, world, port, seed, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rnd = random.Random(seed)
    n, M, steps = 4, 2, 3
    N = n * world
    # global rows: distinct identities, different lengths
    g_rows = [[gid * 1000 + k for k in range(3 + gid % 3)] for gid in range(N)]
    ctx = MockCtx(g_rows[rank * n:(rank + 1) * n])
    for s in range(steps):
        scores = [rnd.randint(0, 3) / 4 for _ in range(N)]   # same stream on every rank
        local = torch.tensor(scores[rank * n:(rank + 1) * n], dtype=torch.float32)
        parent = select_fork_global(ctx, 0, local, M)
        _, want = select_survivors(scores, M)
        assert parent == want
        g_rows = [list(g_rows[p]) for p in want]              # single-rank reference fork
        for i in range(n):                                    # every beam appends a token
            gid = rank * n + i
            ctx.rows[i].append(10_000 * (s + 1) + gid)
        g_rows = [r + [10_000 * (s + 1) + gid] for gid, r in enumerate(g_rows)]
    gathered = [None] * world
    dist.all_gather_object(gathered, ctx.rows)
    if rank == 0:
        out.put((sum(gathered, []), g_rows))
    dist.destroy_process_group()


def test_gloo_world2_select_fork_global():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + random.Random(os.getpid()).randint(0, 2000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 7, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, want = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == want
