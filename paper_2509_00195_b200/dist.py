"""Multi-GPU sharding of the beam-step hot path.

Two partitionings, one process per GPU:

* independent requests (C4): request r -> rank r mod G, each rank its own
  libtts context; no collective on the data path (``shard_requests``);
* one request whose N beams span G ranks (C5): rank k holds global beam ids
  [k*n, (k+1)*n), n = N / G, in DFS order.  Per TTS step the only exchange is
  an all-gather of the N scores (4 B each) and beam lengths, after which every
  rank runs the same global selection (libtts ``tts_beam_select_global``,
  ledger C19: the global id is the tie-break index) and the same deterministic
  placement (child gid c -> rank c // n; the children of one survivor are
  consecutive, so a rank's beams stay a DFS-ordered run).  A child whose
  parent lives on another rank receives the parent's lineage (all its K/V):
  the owner exports it, NCCL point-to-point moves it over NVLink, the
  destination imports it into a spare row, then every rank forks its rows by
  an explicit parent map (``tts_beam_fork_map``).

``migration_plan`` is pure and identical on every rank; the drivers below run
it either over ``torch.distributed`` (NCCL on GPUs, gloo in CPU tests) or over
G contexts in one process ("fake ranks").
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Sequence, Tuple

import torch


def shard_requests(n_requests: int, world: int, rank: int) -> List[int]:
    """C4: request r -> rank r mod G."""
    return [r for r in range(n_requests) if r % world == rank]


@dataclass
class RankPlan:
    local_parent: List[int]                      # child (local index) -> local row after imports
    imports: List[Tuple[int, int]] = field(default_factory=list)   # (parent gid, spare row), ascending gid
    exports: List[Tuple[int, int]] = field(default_factory=list)   # (parent gid, destination rank)


def migration_plan(parent_gid: Sequence[int], world: int) -> List[RankPlan]:
    """Placement + lineage migration for one global fork (identical on all ranks)."""
    N = len(parent_gid)
    assert N % world == 0
    n = N // world
    plans = [RankPlan(local_parent=[]) for _ in range(world)]
    for r in range(world):
        children = range(r * n, (r + 1) * n)
        need = sorted({parent_gid[c] for c in children if parent_gid[c] // n != r})
        slot = {p: n + k for k, p in enumerate(need)}
        plans[r].local_parent = [parent_gid[c] % n if parent_gid[c] // n == r else slot[parent_gid[c]]
                                 for c in children]
        plans[r].imports = [(p, slot[p]) for p in need]
        for p in need:
            plans[p // n].exports.append((p, r))
    for pl in plans:
        pl.exports.sort()
    return plans


def transfers(plans: List[RankPlan], world: int) -> List[Tuple[int, int, int]]:
    """Global ordered list of (parent gid, src rank, dst rank)."""
    n_exp = []
    for s, pl in enumerate(plans):
        for p, d in pl.exports:
            n_exp.append((p, s, d))
    return sorted(n_exp)


# ---------------------------------------------------------------------------
# torch.distributed driver (one process per GPU)

def select_fork_global(ctx, req: int, local_scores: torch.Tensor, width_m: int, group=None):
    """One global fork of request `req` whose beams span the ranks of `group`.

    ctx must provide the libtts context methods (``paper_2509_00195_b200.tts.Context``
    on GPUs; the CPU tests pass a mock with the same surface).  Returns the
    global parent map (list, new gid -> old gid)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = local_scores.numel()
    dev = local_scores.device
    # 1. all-gather scores and lengths (4 B + 4 B per beam)
    sc = [torch.empty_like(local_scores) for _ in range(world)]
    dist.all_gather(sc, local_scores.contiguous(), group=group)
    lens_local = torch.as_tensor(ctx.tts_seq_lens_host(req)[:n].copy(), dtype=torch.int32, device=dev)
    ln = [torch.empty_like(lens_local) for _ in range(world)]
    dist.all_gather(ln, lens_local, group=group)
    scores_all = torch.cat(sc)
    lens_all = torch.cat(ln).cpu().tolist()
    # 2. global selection, identical on every rank
    parent = torch.empty(n * world, dtype=torch.int32, device=dev)
    ctx.tts_beam_select_global(scores_all, width_m, parent)
    parent = parent.cpu().tolist()
    # 3. placement and migration plan
    plans = migration_plan(parent, world)
    me = plans[rank]
    # 4. lineage exchange (grouped point-to-point: no ordering deadlock)
    ops, recv_bufs = [], []
    for p, d in me.exports:
        buf = ctx.lineage_buffer(lens_all[p])
        ctx.tts_lineage_export(req, p % n, buf)
        ops.append(dist.P2POp(dist.isend, buf, d, group=group))
    for p, slot in me.imports:
        buf = ctx.lineage_buffer(lens_all[p])
        recv_bufs.append((slot, lens_all[p], buf))
        ops.append(dist.P2POp(dist.irecv, buf, p // n, group=group))
    if ops:
        ctx.sync()
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    for slot, length, buf in recv_bufs:
        ctx.tts_lineage_import(req, slot, length, buf)
    # 5. local fork by map
    ctx.tts_beam_fork_map(req, me.local_parent)
    return parent


# ---------------------------------------------------------------------------
# fake-rank driver: G contexts in one process (single-GPU test of the real kernels)

def select_fork_global_fake(ctxs: Sequence, req: int, local_scores: Sequence[torch.Tensor], width_m: int):
    world = len(ctxs)
    n = local_scores[0].numel()
    scores_all = torch.cat([s.to(local_scores[0].device) for s in local_scores])
    lens_all = []
    for c in ctxs:
        lens_all += list(c.tts_seq_lens_host(req)[:n])
    parents = []
    for c in ctxs:
        par = torch.empty(n * world, dtype=torch.int32, device=scores_all.device)
        c.tts_beam_select_global(scores_all, width_m, par)
        parents.append(par.cpu().tolist())
    assert all(p == parents[0] for p in parents), "global selection differs across ranks"
    parent = parents[0]
    plans = migration_plan(parent, world)
    staged: Dict[Tuple[int, int], torch.Tensor] = {}
    for p, s, d in transfers(plans, world):
        buf = ctxs[s].lineage_buffer(lens_all[p])
        ctxs[s].tts_lineage_export(req, p % n, buf)
        staged[(p, d)] = buf
    for d, pl in enumerate(plans):
        for p, slot in pl.imports:
            ctxs[d].tts_lineage_import(req, slot, lens_all[p], staged[(p, d)])
    for d, pl in enumerate(plans):
        ctxs[d].tts_beam_fork_map(req, pl.local_parent)
    return parent
