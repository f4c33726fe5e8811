"""Multi-GPU plumbing of the beam-step hot path.  Nothing here
computes the method: selection, placement, lineage migration and the fork
run inside libtts (tts_beam_select_fork_global); this module only moves the
bytes libtts asks it to move, or sets up the NCCL communicator libtts owns.

Two partitionings, one process per GPU:

* independent requests (C4): request r -> rank r mod G, each rank its own
  libtts context; no collective on the data path (``shard_requests``);
* one request whose N beams span G ranks (C5): ``nccl_comm`` gives every
  rank's context the NCCL communicator (unique id broadcast over
  torch.distributed), ``tts_span_init`` declares the request spanning, and
  ``tts_beam_select_fork_global`` runs the cross-rank step.

Host transports (``tts_comm_init_host``) for testing the same library path
without NCCL: ``GlooTransport`` (a torch.distributed gloo group: processes,
possibly sharing one GPU) and ``ThreadGroup`` (threads of one process acting
as ranks, SURVEY 4 item 5a "fake ranks").
"""
from __future__ import annotations

import threading
from typing import Dict, List, Sequence, Tuple

import torch


def shard_requests(n_requests: int, world: int, rank: int) -> List[int]:
    """C4: request r -> rank r mod G."""
    return [r for r in range(n_requests) if r % world == rank]


def equal_caps(n_global: int, world: int) -> List[int]:
    """Beams per rank for an equal-count initial cut (every beam holds only the
    prompt at install, so equal counts are equal bytes)."""
    base, extra = divmod(n_global, world)
    return [base + (1 if r < extra else 0) for r in range(world)]


def nccl_comm(ctx, group=None, stage_bytes: int = 1 << 30) -> torch.Tensor:
    """Joins ctx to an NCCL communicator over the ranks of `group` (rank 0
    creates the unique id, torch.distributed broadcasts it).  Returns the
    device staging buffer libtts borrows (keep it alive)."""
    import torch.distributed as dist
    from .tts import comm_unique_id
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    obj = [comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    stage = torch.empty(stage_bytes, dtype=torch.uint8, device=ctx.device)
    ctx.tts_comm_init(obj[0], world, rank, stage)
    return stage


class GlooTransport:
    """Host transport over a torch.distributed (gloo) group: byte buffers as
    CPU uint8 tensors."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)

    def allgather(self, data: bytes, nbytes: int) -> bytes:
        t = torch.frombuffer(bytearray(data), dtype=torch.uint8)
        out = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return b"".join(o.numpy().tobytes() for o in out)

    def sendrecv(self, sends: Sequence[Tuple[int, bytes]], recvs: Sequence[Tuple[int, int]]) -> List[bytes]:
        ops, bufs = [], []
        for dst, data in sends:
            ops.append(self.dist.P2POp(self.dist.isend, torch.frombuffer(bytearray(data), dtype=torch.uint8), dst,
                                       group=self.group))
        for src, n in recvs:
            b = torch.empty(n, dtype=torch.uint8)
            bufs.append(b)
            ops.append(self.dist.P2POp(self.dist.irecv, b, src, group=self.group))
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()
        return [b.numpy().tobytes() for b in bufs]


class ThreadGroup:
    """G threads of one process acting as ranks: ``transport(r)`` is rank r's
    host transport (collective calls rendezvous on a barrier)."""

    def __init__(self, world: int):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots: List[bytes] = [b""] * world
        self.mail: Dict[Tuple[int, int], List[bytes]] = {}
        self.lock = threading.Lock()

    def transport(self, rank: int) -> "_ThreadTransport":
        return _ThreadTransport(self, rank)


class _ThreadTransport:
    def __init__(self, g: ThreadGroup, rank: int):
        self.g, self.rank = g, rank

    def allgather(self, data: bytes, nbytes: int) -> bytes:
        g = self.g
        g.slots[self.rank] = bytes(data)
        g.barrier.wait()
        out = b"".join(g.slots)
        g.barrier.wait()
        return out

    def sendrecv(self, sends, recvs) -> List[bytes]:
        g = self.g
        with g.lock:
            for dst, data in sends:
                g.mail.setdefault((self.rank, dst), []).append(bytes(data))
        g.barrier.wait()
        got = []
        with g.lock:
            for src, n in recvs:
                m = g.mail[(src, self.rank)].pop(0)
                assert len(m) == n
                got.append(m)
        g.barrier.wait()
        return got
