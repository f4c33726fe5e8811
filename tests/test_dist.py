"""Multi-rank host logic on CPU: libtts's placement rule (a
host-only C-ABI call, no GPU) against the oracle rank model, and the byte
transports the library drives (gloo at world size 2 in two processes;
threads of one process)."""
import os
import random
import socket
import threading

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.ranks import placement as oracle_placement
from oracle.select import select_survivors
from paper_2509_00195_b200.dist import ThreadGroup, equal_caps, shard_requests


def test_shard_requests_partition():
    for G in (1, 2, 4, 8):
        parts = [shard_requests(64, G, r) for r in range(G)]
        assert sorted(sum(parts, [])) == list(range(64))
        assert max(map(len, parts)) - min(map(len, parts)) <= 1


def test_equal_caps():
    assert equal_caps(512, 8) == [64] * 8
    assert equal_caps(10, 4) == [3, 3, 2, 2]


@pytest.fixture(scope="module")
def lib():
    from paper_2509_00195_b200 import build, tts
    build.build()
    return tts.load()


@pytest.mark.parametrize("seed", range(40))
def test_libtts_placement_equals_oracle(lib, seed):
    """tts_span_placement (C++, identical on every rank) against
    oracle.ranks.placement (written from 8(e) step 3)."""
    from paper_2509_00195_b200.tts import span_placement
    rnd = random.Random(seed)
    G = rnd.choice([1, 2, 3, 4, 8])
    caps = [rnd.randint(1, 9) for _ in range(G)]
    N = sum(caps)
    M = rnd.choice([m for m in (1, 2, 4, 8) if N % m == 0])
    _, parent = select_survivors([rnd.randint(0, 5) / 5 for _ in range(N)], M)
    old_rank = sum([[r] * caps[r] for r in range(G)], [])
    rnd.shuffle(old_rank)
    assert span_placement(parent, old_rank, caps) == oracle_placement(parent, old_rank, caps)


def test_libtts_placement_rejects_bad_capacities(lib):
    from paper_2509_00195_b200.tts import TTSError, span_placement
    with pytest.raises(TTSError):
        span_placement([0, 0, 1, 1], [0, 0, 1, 1], [2, 1])      # sum != N
    with pytest.raises(TTSError):
        span_placement([0, 0, 5, 1], [0, 0, 1, 1], [2, 2])      # parent out of range


def test_thread_group_transport():
    G = 4
    grp = ThreadGroup(G)
    out = {}

    def work(r):
        t = grp.transport(r)
        ag = t.allgather(bytes([r] * 3), 3)
        sends = [((r + 1) % G, f"to{(r + 1) % G}from{r}".encode()), ((r + 2) % G, b"x" * r)]
        recvs = [((r - 1) % G, len(f"to{r}from{(r - 1) % G}")), ((r - 2) % G, (r - 2) % G)]
        got = t.sendrecv(sends, recvs)
        out[r] = (ag, got)

    th = [threading.Thread(target=work, args=(r,)) for r in range(G)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    for r in range(G):
        ag, got = out[r]
        assert ag == b"".join(bytes([q] * 3) for q in range(G))
        assert got[0] == f"to{r}from{(r - 1) % G}".encode() and got[1] == b"x" * ((r - 2) % G)


def _gloo_transport_worker(rank, world, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2509_00195_b200.dist import GlooTransport
        t = GlooTransport()
        ag = t.allgather(bytes([7 + rank] * 5), 5)
        assert ag == bytes([7] * 5) + bytes([8] * 5)
        other = 1 - rank
        sends = [(other, f"lineage-{rank}-a".encode()), (other, b"B" * (100 + rank))]
        recvs = [(other, len(f"lineage-{other}-a")), (other, 100 + other)]
        got = t.sendrecv(sends, recvs)
        assert got == [f"lineage-{other}-a".encode(), b"B" * (100 + other)]
        assert t.sendrecv([], []) == []
    finally:
        dist.destroy_process_group()


def test_gloo_transport_world2():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_gloo_transport_worker, args=(2, port), nprocs=2, join=True)
