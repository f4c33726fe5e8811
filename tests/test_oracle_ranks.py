"""Pins for oracle.ranks (CPU): the rank model of a request whose beams span G
GPUs (ledger C19/C20) against the single-rank oracle (which the
other oracle tests pin to the paper), a hand-derived two-rank migration, and
the placement rule's defining properties."""
import random

import numpy as np
import pytest

from oracle.block_table import BlockTableSim
from oracle.ranks import SpanModel, placement, rank_plans
from oracle.select import select_survivors


def test_hand_derived_two_rank_migration():
    """N = 4, M = 2, two ranks of capacity 2, prompt 32 (pages 0, 1 on each
    rank's own allocator), one 16-token step.  Scores [0.9, 0.8, 0.1, 0.2]
    keep gids {0, 1}, both on rank 0: children 0, 1 stay there (capacity 2),
    children 2, 3 (parent 1) overflow to rank 1, which imports gid 1's whole
    48-token lineage into spare row 2 (fresh pages 4, 5, 6, after its pages
    0-3), then forks both rows from it; every old page of rank 1 drops to 0."""
    m = SpanModel(N=4, caps=[2, 2], num_pages=16, P=16, prompt_len=32)
    for t in range(16):
        m.append([1, 1, 1, 1], [("d", 0, t, g) for g in range(4)])
    assert m.sims[0].tables[0] == [[0, 1, 2], [0, 1, 3]]
    assert m.sims[1].tables[0] == [[0, 1, 2], [0, 1, 3]]
    rec = m.fork([0.9, 0.8, 0.1, 0.2], 2)
    assert rec.parent_gid == [0, 0, 1, 1]
    assert rec.child_rank == [0, 0, 1, 1]
    assert rec.plans[1].imports == [1] and rec.plans[1].parent_rows == [2, 2]
    assert rec.plans[0].imports == [] and rec.plans[0].parent_rows == [0, 0]
    assert rec.tables[0] == [[0, 1, 2], [0, 1, 2]]
    assert rec.tables[1] == [[4, 5, 6], [4, 5, 6]]
    assert [p for p, r in enumerate(rec.ref[1]) if r] == [4, 5, 6] and rec.ref[1][4] == 2
    assert rec.free[1] == [p for p in range(16) if p not in (4, 5, 6)]
    assert rec.free[0] == [p for p in range(16) if p not in (0, 1, 2)]
    assert m.gids == [[0, 1], [2, 3]]
    # children inherit the parent's prefix: gid 2 and 3 read gid 1's tokens
    want = [("p", 0, i) for i in range(32)] + [("d", 0, t, 1) for t in range(16)]
    assert m.gather(2) == want and m.gather(3) == want


@pytest.mark.parametrize("seed", range(30))
def test_placement_rule_properties(seed):
    rnd = random.Random(seed)
    G = rnd.choice([2, 3, 4, 8])
    caps = [rnd.randint(1, 6) for _ in range(G)]
    N = sum(caps)
    M = rnd.choice([m for m in (1, 2, 3, 4, 8) if N % m == 0])
    scores = [rnd.randint(0, 7) / 8 for _ in range(N)]
    _, parent = select_survivors(scores, M)
    old_rank = sum([[r] * caps[r] for r in range(G)], [])
    rnd.shuffle(old_rank)
    cr = placement(parent, old_rank, caps)
    assert [cr.count(r) for r in range(G)] == caps
    for c in range(N):
        pr = old_rank[parent[c]]
        stayed_before = sum(1 for x in range(c) if cr[x] == pr and old_rank[parent[x]] == pr)
        if cr[c] != pr:
            assert stayed_before == caps[pr], "a child left its parent's rank while capacity remained"
    over = [cr[c] for c in range(N) if cr[c] != old_rank[parent[c]]]
    assert over == sorted(over), "overflow children go to the lowest rank with free capacity, in gid order"


def test_one_rank_reduces_to_single_gpu_fork():
    """G = 1: no migration; fork_map with the select_survivors parent map is
    the single-rank fork (BlockTableSim.fork): same tables, refcounts, free set."""
    rnd = random.Random(3)
    for trial in range(10):
        N, M, P = 8, rnd.choice([2, 4]), 16
        m = SpanModel(N=N, caps=[N], num_pages=200, P=P, prompt_len=rnd.choice([0, 7, 16, 37]))
        ref = BlockTableSim(200, P)
        ref.init_request(0, N, m.sims[0].lens[0][0], [("p", 0, i) for i in range(m.sims[0].lens[0][0])])
        for step in range(4):
            for t in range(rnd.randint(1, 40)):
                act = [rnd.random() < 0.8 for _ in range(N)]
                ids = [("d", 0, step * 100 + t, g) for g in range(N)]
                m.append(act, ids)
                ref.append([0], [act], [ids])
            sc = [rnd.randint(0, 4) / 4 for _ in range(N)]
            rec = m.fork(sc, M)
            ref.fork([0], [sc], M)
            assert rec.tables[0] == ref.tables[0] and rec.lens[0] == ref.lens[0]
            assert rec.ref[0] == ref.ref and rec.free[0] == ref.free_set()


@pytest.mark.parametrize("seed", range(12))
def test_span_model_matches_single_rank_oracle(seed):
    """Any G and capacities: survivors and every beam's token sequence (read
    through the owning rank's pages) equal the single-rank oracle's at every
    fork (ledger C20); each rank's refcounts are the number of its tables
    holding the page and its free set is the complement (C8)."""
    rnd = random.Random(100 + seed)
    G = rnd.choice([2, 4, 8])
    per = rnd.choice([1, 2, 4])
    caps = [per] * G if rnd.random() < 0.5 else [rnd.randint(1, 2 * per) for _ in range(G)]
    N = sum(caps)
    M = rnd.choice([m for m in (2, 4, 8) if N % m == 0] or [1])
    P = 16
    prompt = rnd.choice([0, 5, 16, 37])
    m = SpanModel(N=N, caps=caps, num_pages=4000, P=P, prompt_len=prompt)
    ref = BlockTableSim(4000 * G, P)
    ref.init_request(0, N, prompt, [("p", 0, i) for i in range(prompt)])
    t = 0
    for step in range(5):
        for _ in range(rnd.randint(1, 30)):
            act = [rnd.random() < 0.85 for _ in range(N)]
            ids = [("d", 0, t, g) for g in range(N)]
            m.append(act, ids)
            ref.append([0], [act], [ids])
            t += 1
        sc = [rnd.randint(0, 5) / 5 for _ in range(N)]
        rec = m.fork(sc, M)
        par = ref.fork([0], [sc], M)[0]
        assert rec.parent_gid == par
        assert m.lens_by_gid() == ref.lens[0]
        for g in range(N):
            assert m.gather(g) == ref.gather(0, g)
        for r in range(G):
            tables = rec.tables[r]
            cnt = np.zeros(4000, dtype=int)
            for row, ln in zip(tables, rec.lens[r]):
                assert len(row) == -(-ln // P)
                for p in row:
                    cnt[p] += 1
            assert cnt.tolist() == rec.ref[r]
            assert rec.free[r] == [p for p in range(4000) if cnt[p] == 0]
        # a rank's beams are in ascending gid, so every subtree's beams on a rank are adjacent rows
        assert all(gs == sorted(gs) for gs in m.gids)


def test_dedup_hand_example():
    """f4: N = 4, M = 2, ranks [2, 2], a 32-token prompt and a 16-token step,
    then a second step.  Fork 1 keeps gids {0, 1} (both on rank 0): rank 1
    imports gid 1's 48-token lineage; its beams share only the prompt with it
    (2 full pages), so the import reuses rank 1's own prompt pages 0, 1 and
    allocates one page for the step's tokens -- 16 tokens cross, not 48."""
    m = SpanModel(N=4, caps=[2, 2], num_pages=16, P=16, prompt_len=32, dedup=True)
    for t in range(16):
        m.append([1, 1, 1, 1], [("d", 0, t, g) for g in range(4)])
    rec = m.fork([0.9, 0.8, 0.1, 0.2], 2)
    assert rec.tables[1] == [[0, 1, 4], [0, 1, 4]]
    assert m.migrated_tokens == 16 and m.deduped_tokens == 32
    assert m.gather(2) == [("p", 0, i) for i in range(32)] + [("d", 0, t, 1) for t in range(16)]


@pytest.mark.parametrize("seed", range(12))
def test_dedup_preserves_sequences_and_saves_bytes(seed):
    """Deduplication changes page ids, never what any beam reads: every beam's
    token sequence equals the non-dedup model's at every fork; no more
    tokens cross than without it; refcounts = table counts."""
    rnd = random.Random(300 + seed)
    G = rnd.choice([2, 4])
    caps = [rnd.choice([2, 4])] * G
    N = sum(caps)
    M = rnd.choice([m for m in (2, 4) if N % m == 0])
    prompt = rnd.choice([16, 37, 64])
    a = SpanModel(N=N, caps=caps, num_pages=4000, P=16, prompt_len=prompt, dedup=True)
    b = SpanModel(N=N, caps=caps, num_pages=4000, P=16, prompt_len=prompt, dedup=False)
    t = 0
    for step in range(4):
        for _ in range(rnd.randint(8, 40)):
            act = [rnd.random() < 0.9 for _ in range(N)]
            for mm in (a, b):
                mm.append(act, [("d", 0, t, g) for g in range(N)])
            t += 1
        sc = [rnd.randint(0, 3) / 3 for _ in range(N)]
        ra, rb = a.fork(sc, M), b.fork(sc, M)
        assert ra.parent_gid == rb.parent_gid and ra.child_rank == rb.child_rank
        for g in range(N):
            assert a.gather(g) == b.gather(g)
        for r in range(G):
            cnt = np.zeros(4000, dtype=int)
            for row in ra.tables[r]:
                for p in row:
                    cnt[p] += 1
            assert cnt.tolist() == ra.ref[r]
    assert a.migrated_tokens <= b.migrated_tokens
    assert a.migrated_tokens + a.deduped_tokens == b.migrated_tokens
