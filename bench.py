#!/usr/bin/env python
"""Benchmark of the FlashTTS beam-step hot path on B200 (libtts through its C-ABI).

One bench *step* = one complete TTS run of the configuration for every
request a rank holds: install on the prompt, every decode iteration (append +
prefix-shared attention over all L layers), a select + fork after every TTS
step but the last, release.  All SURVEY 8(a) rows are inside the timed region.

Workload (BASELINE.json configs; the metric names none, so N = 1 runs the
largest single-GPU configuration): default at N = 1 is C3 (configs[2],
Qwen2.5-Math-7B attention shape, N = 64, M = 4, 4k-token chains; its unique KV
per position, ~1.4 GB, is >> the 126 MB L2, so consecutive calls find nothing
of theirs in L2 -- SURVEY 8(d) pitfall 1 "inputs larger than L2").  C2 and the
other configs via --config; C2 rotates --rotate independent requests (one per
call) so that the reuse distance of a page spans >= 2x L2.
Multi-GPU: one process per GPU.  Default at N > 1 is C4 (64 concurrent
requests, request r -> rank r mod N, no data-path collective, "scaling":
"strong"); --config C5 spreads one request's 512 beams over the ranks (NCCL
all-gather of scores + lineage migration per step).  `--gpus N` without
torchrun re-launches itself under torch.distributed.run with N processes.

--impl reference times the CPU oracle (the only reference this paper-only
task has) on the host cores, on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import workload  # noqa: E402

METRIC = "beam-steps/s and HBM GB/s (unique KV) vs roofline at 1/2/4/8 B200"
UNIT = "beam-steps/s"
DEFAULT_ROTATE = {"C1": 64, "C2": 32, "C3": 1, "C4": 1, "C5": 1}
DEFAULT_PER_CALL = {"C1": 1, "C2": 32, "C3": 1, "C4": 1, "C5": 1}  # C2: all 32 rotated requests batched per call (same requests and tokens); measured 4 -> 0.62, 8 -> 0.71, 16 -> 0.75, 32 -> 0.78 of the copy peak
HBM_SPEC_GBS = 8000.0  # north_star "~8 TB/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="libtts", choices=["libtts", "reference"])
    ap.add_argument("--config", default=None, choices=list(workload.CONFIGS),
                    help="default: C3 at N = 1, C4 at N > 1")
    ap.add_argument("--rotate", type=int, default=0)
    ap.add_argument("--per-call", type=int, default=0,
                    help="requests of the rotation per decode call (fixed-step configs; default per config)")
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=18.0)
    ap.add_argument("--dump-call-bytes", default="")
    ap.add_argument("--requests", type=int, default=0, help="override R of the straggler batch (C4)")
    ap.add_argument("--tts-steps", type=int, default=0, help="override the number of TTS steps (shorter chains)")
    ap.add_argument("--pages-per-request", type=int, default=0,
                    help="page-pool budget per request (default: exact bound for fixed steps, 6000 for C4)")
    return ap.parse_args()


def resolve_config(args, ws):
    return args.config or ("C3" if ws == 1 else "C4")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_spawn(args):
    """`--gpus N` (N > 1) outside torchrun: re-launch under torch.distributed.run,
    one process per GPU; fail loudly if the box has fewer GPUs."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    if args.impl == "libtts":
        have = torch.cuda.device_count()
        if have < args.gpus:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, this box has {have}\n")
            sys.exit(2)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def dist_init(n):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws != n:
        raise SystemExit(f"bench.py: WORLD_SIZE={ws} but --gpus {n}")
    if ws > 1:
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def allmax(x, ws, dev):
    if ws == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allsum(x, ws, dev):
    if ws == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    def __init__(self, dev_index):
        self.p = None
        self.path = f"/tmp/tts_clocks_{os.getpid()}.csv"
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(dev_index), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        rows = []
        for ln in open(self.path):
            f = [x.strip() for x in ln.split(",")]
            if len(f) >= 7 and f[0].isdigit():
                rows.append(f)
        if not rows:
            return None
        sm = [int(r[0]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        under = [s for s in sm if s > 500] or sm
        return {"sm_mhz": statistics.median(under), "sm_max_mhz": int(rows[0][1]), "reasons": reasons,
                "samples": len(sm)}


# ---------------------------------------------------------------------------
class IOPipe:
    """Host <-> device traffic of a serving loop that feeds the C-ABI from host
    buffers: each call's q/k/v are copied H2D (pinned, on a copy stream) into
    one of two device slots while the previous call computes, and each call's
    output is copied D2H (pinned, on a second copy stream) once the call has
    run, so the next call's kernels overlap both copies."""

    def __init__(self, like_in, like_out, dev):
        self.slots = [tuple(torch.empty_like(t) for t in like_in) for _ in range(2)]
        self.outs = [torch.empty_like(like_out) for _ in range(2)]
        self.host_out = [torch.empty(like_out.shape, dtype=like_out.dtype).pin_memory() for _ in range(2)]
        self.h2d = torch.cuda.Stream(dev)
        self.d2h = torch.cuda.Stream(dev)
        self.ready = [torch.cuda.Event() for _ in range(2)]
        self.used = [torch.cuda.Event() for _ in range(2)]
        self.out_free = [torch.cuda.Event() for _ in range(2)]
        self.i = 0
        self.dev = dev
        self.d2h_bytes = 0

    def stage(self, hq, hk, hv):
        s = self.i & 1
        with torch.cuda.stream(self.h2d):
            self.h2d.wait_event(self.used[s])  # the call that last read this slot has run
            q, k, v = self.slots[s]
            q.copy_(hq, non_blocking=True)
            k.copy_(hk, non_blocking=True)
            v.copy_(hv, non_blocking=True)
            self.ready[s].record(self.h2d)
        cur = torch.cuda.current_stream(self.dev)
        cur.wait_event(self.ready[s])
        cur.wait_event(self.out_free[s])  # this slot's previous output has reached the host
        return q, k, v, self.outs[s]

    def release(self):
        s = self.i & 1
        self.used[s].record(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(self.d2h):
            self.d2h.wait_event(self.used[s])
            self.host_out[s].copy_(self.outs[s], non_blocking=True)
            self.out_free[s].record(self.d2h)
        self.d2h_bytes += self.outs[s].numel() * self.outs[s].element_size()
        self.i += 1

    def drain(self):
        torch.cuda.current_stream(self.dev).wait_stream(self.d2h)


# ---------------------------------------------------------------------------
class Bench:
    """Drives one rank's requests through libtts with minimal host overhead."""

    def __init__(self, cfg, greqs, dev_index, ring=8, pages_per_request=0, per_call=1):
        from paper_2509_00195_b200 import build
        build.build()
        from paper_2509_00195_b200.runner import tts_config, Inputs
        from paper_2509_00195_b200.tts import Context
        self.cfg = cfg
        self.greqs = list(greqs)
        self.n = len(self.greqs)
        self.tcfg = tts_config(cfg, self.n, num_pages=(pages_per_request * self.n + 64) if pages_per_request else None)
        self.ctx = Context(self.tcfg, dev_index)
        self.lib = self.ctx.lib
        self.h = self.ctx.h
        self.dev = self.ctx.device
        self.inp = Inputs(cfg, self.dev)
        self.scale = ctypes.c_float(1.0 / math.sqrt(cfg.d))
        self.batched = cfg.step_len == 0  # straggler configs: one call per iteration for all requests
        # fixed-step configs: `per_call` consecutive requests of the rotation per
        # decode call (the C-ABI's n_req; 1 = one request per call)
        per_call = self.n if self.batched else max(1, min(per_call, self.n))
        self.per_call = per_call
        self.ring = []
        for i in range(ring):
            q, k, v = self.inp.step(10_000 + i, self.greqs[:per_call])
            self.ring.append((q, k, v))
        self.out = torch.empty(cfg.L, per_call, cfg.N, cfg.Hq, cfg.d, dtype=torch.float32, device=self.dev)
        self.prompt = [self.inp.prompt_kv(r) for r in self.greqs]
        self.sched = list(workload.schedule(cfg, self.greqs))
        self.scores = {}
        for it in self.sched:
            for r, s in it.forks:
                self.scores[(r, s)] = self.inp.scores(r, s).contiguous()
        self.local = {r: i for i, r in enumerate(self.greqs)}
        self.req_arr = {i: (ctypes.c_int32 * 1)(i) for i in range(self.n)}
        # request chunks of a decode call (fixed-step configs: every request is live at every iteration)
        self.chunks = [[self.local[r] for r in self.greqs[i:i + per_call]] for i in range(0, self.n, per_call)]
        self.chunk_arr = [(ctypes.c_int32 * len(ch))(*ch) for ch in self.chunks]
        self.parent = torch.empty(self.n, cfg.N, dtype=torch.int32, device=self.dev)
        self.beam_steps = sum(int(a.sum()) for it in self.sched for a in it.active)
        self.stream = self.ctx.stream
        self.ncall = 0
        self.n_calls = sum(1 if self.batched else -(-len(it.reqs) // per_call) for it in self.sched)
        torch.cuda.synchronize(self.dev)

    def _chk(self, code, what):
        if code != 0:
            from paper_2509_00195_b200.tts import TTSError
            raise TTSError(code, what)

    def run_step(self, stats_accum=None, e2e=None, seg=None, forks=None):
        """One full run of every request.  e2e: dict with the pinned host input
        ring and the IOPipe.  seg: list receiving one CUDA event pair (on the
        launching stream) per run of consecutive decode calls between two forks
        (install / release excluded).  forks: list receiving one event pair
        around every tts_beam_select_fork call."""
        c = self.cfg
        open_ev = None
        lib, h, st = self.lib, self.h, self.stream
        cur = torch.cuda.current_stream(self.dev)
        for r in self.greqs:
            k, v = self.prompt[self.local[r]]
            self._chk(lib.tts_block_table_init_request(h, self.local[r], c.N, c.prompt, k.data_ptr(),
                                                       v.data_ptr(), st), "init")
        nr = len(self.ring)
        ptrs = [(ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(k.data_ptr()), ctypes.c_void_p(v.data_ptr()))
                for q, k, v in self.ring]
        outp = ctypes.c_void_p(self.out.data_ptr())
        decode = lib.tts_decode_step
        for it in self.sched:
            q, k, v = self.ring[it.t % nr]
            out = self.out
            if seg is not None and open_ev is None:
                open_ev = torch.cuda.Event(enable_timing=True)
                open_ev.record(cur)
            if e2e is None and not self.batched and stats_accum is None:
                # hot loop: one C-ABI call per request and position, arguments pre-marshalled
                qp, kp, vp = ptrs[it.t % nr]
                for ch, arr in zip(self.chunks, self.chunk_arr):
                    rc = decode(h, len(ch), arr, None, kp, vp, qp, self.scale, outp, st)
                    if rc:
                        self._chk(rc, "decode_step")
            else:
                if e2e is not None:
                    hq, hk, hv = e2e["ring"][it.t % nr]
                if self.batched:
                    if e2e is not None:
                        q, k, v, out = e2e["pipe"].stage(hq, hk, hv)
                    loc = [self.local[r] for r in it.reqs]
                    arr = (ctypes.c_int32 * len(loc))(*loc)
                    act = np.ascontiguousarray(np.stack(it.active), dtype=np.uint8)
                    self._chk(lib.tts_decode_step(h, len(loc), arr, act.ctypes.data_as(ctypes.c_void_p),
                                                  k.data_ptr(), v.data_ptr(), q.data_ptr(), self.scale,
                                                  out.data_ptr(), st), "decode_step")
                    if e2e is not None:
                        e2e["pipe"].release()
                    if stats_accum is not None:
                        self._chk(lib.tts_block_table_stats(h, len(loc), arr, act.ctypes.data_as(ctypes.c_void_p),
                                                            stats_accum[self.ncall].data_ptr(), st), "stats")
                        self.ncall += 1
                else:
                    for ch, arr in zip(self.chunks, self.chunk_arr):
                        if e2e is not None:  # every call's q/k/v come from the host, its output goes back
                            q, k, v, out = e2e["pipe"].stage(hq, hk, hv)
                        self._chk(lib.tts_decode_step(h, len(ch), arr, None, k.data_ptr(), v.data_ptr(),
                                                      q.data_ptr(), self.scale, out.data_ptr(), st), "decode_step")
                        if e2e is not None:
                            e2e["pipe"].release()
                        if stats_accum is not None:
                            self._chk(lib.tts_block_table_stats(h, len(ch), arr, None,
                                                                stats_accum[self.ncall].data_ptr(), st), "stats")
                            self.ncall += 1
            if it.forks or (seg is not None and it is self.sched[-1]):
                if seg is not None:
                    e_end = torch.cuda.Event(enable_timing=True)
                    e_end.record(cur)
                    seg.append((open_ev, e_end))
                    open_ev = None
            if it.forks:
                loc = [self.local[r] for r, _ in it.forks]
                arr = (ctypes.c_int32 * len(loc))(*loc)
                sc = torch.stack([self.scores[(r, s)] for r, s in it.forks]) if len(loc) > 1 else \
                    self.scores[it.forks[0]].view(1, -1)
                if e2e is not None:  # the PRM scores come from the host, the parent maps go back
                    sc = sc.cpu().pin_memory().to(self.dev, non_blocking=True)
                if forks is not None:
                    f0 = torch.cuda.Event(enable_timing=True)
                    f0.record(cur)
                self._chk(lib.tts_beam_select_fork(h, len(loc), arr, sc.data_ptr(), c.M,
                                                   self.parent.data_ptr(), st), "select_fork")
                if forks is not None:
                    f1 = torch.cuda.Event(enable_timing=True)
                    f1.record(cur)
                    forks.append((f0, f1))
                if e2e is not None:
                    e2e["d2h"] += self.parent[: len(loc)].numel() * 4
                    e2e["h2d"] += sc.numel() * 4
                    e2e["parents"].append(self.parent[: len(loc)].to("cpu", non_blocking=True))
        if e2e is not None:
            e2e["pipe"].drain()
        for r in self.greqs:
            self._chk(lib.tts_block_table_release_request(h, self.local[r], st), "release")


class SpanBench:
    """C5: one request whose N beams span the G ranks (n = N / G per rank).
    Per decode iteration each rank runs append + attention on its n beams; at
    every step end libtts runs the cross-rank step on every rank
    (tts_beam_select_fork_global over its NCCL communicator: all-gather of
    (score, gid, len), global selection, placement, lineage migration, fork)."""

    def __init__(self, cfg, world, rank, dev_index, ring=8):
        from paper_2509_00195_b200 import build
        build.build()
        from paper_2509_00195_b200.runner import tts_config, Inputs, pages_per_request
        from paper_2509_00195_b200.tts import Context
        self.cfg, self.world, self.rank = cfg, world, rank
        self.dedup = os.environ.get("TTS_SPAN_DEDUP", "1") != "0"  # f4: cross-GPU page deduplication
        self.nl = cfg.N // world
        maxb = 2 * self.nl if world > 1 else cfg.N
        if world == 1:
            pages = pages_per_request(cfg) + 256  # the whole tree on one rank
        else:
            pages = 2 * self.nl * workload.max_pages_per_beam(cfg) + 256  # imported lineages are private copies
        self.tcfg = tts_config(cfg, 1, num_pages=pages, max_beams=maxb)
        self.ctx = Context(self.tcfg, dev_index)
        self.lib, self.h, self.dev = self.ctx.lib, self.ctx.h, self.ctx.device
        self.stage = None
        if world > 1:
            from paper_2509_00195_b200.dist import nccl_comm
            self.stage = nccl_comm(self.ctx, stage_bytes=4 << 30)
        self.inp = Inputs(cfg, self.dev)
        self.scale = ctypes.c_float(1.0 / math.sqrt(cfg.d))
        self.batched = False
        self.greqs = [0]
        self.ring = []
        for i in range(ring):
            q = torch.randn(cfg.L, 1, maxb, cfg.Hq, cfg.d, device=self.dev).to(torch.bfloat16)
            k = torch.randn(cfg.L, 1, maxb, cfg.Hkv, cfg.d, device=self.dev).to(torch.bfloat16)
            v = torch.randn(cfg.L, 1, maxb, cfg.Hkv, cfg.d, device=self.dev).to(torch.bfloat16)
            self.ring.append((q, k, v))
        self.out = torch.empty(cfg.L, 1, maxb, cfg.Hq, cfg.d, dtype=torch.float32, device=self.dev)
        self.prompt = self.inp.prompt_kv(0)
        self.sched = list(workload.schedule(cfg, [0]))
        self.scores = {s: self.inp.scores(0, s).contiguous() for it in self.sched for (_, s) in it.forks}
        self.beam_steps = sum(int(it.active[0][rank * self.nl:(rank + 1) * self.nl].sum()) for it in self.sched)
        self.n_calls = len(self.sched)
        self.ncall = 0
        self.stream = self.ctx.stream
        self.req = (ctypes.c_int32 * 1)(0)
        torch.cuda.synchronize(self.dev)

    def _chk(self, code, what):
        if code != 0:
            from paper_2509_00195_b200.tts import TTSError
            raise TTSError(code, what)

    def run_step(self, stats_accum=None, e2e=None, seg=None, forks=None):
        c, lib, h, st = self.cfg, self.lib, self.h, self.stream
        k, v = self.prompt
        self._chk(lib.tts_block_table_init_request(h, 0, self.nl, c.prompt, k.data_ptr(), v.data_ptr(), st), "init")
        if self.world > 1:
            from paper_2509_00195_b200.dist import equal_caps
            self.ctx.tts_span_init(0, c.N, equal_caps(c.N, self.world), self.dedup)
        nr = len(self.ring)
        open_ev = None
        for it in self.sched:
            q, k, v = self.ring[it.t % nr]
            if seg is not None and open_ev is None:
                open_ev = torch.cuda.Event(enable_timing=True)
                open_ev.record(torch.cuda.current_stream(self.dev))
            out = self.out
            if e2e is not None:
                hq, hk, hv = e2e["ring"][it.t % nr]
                q, k, v, out = e2e["pipe"].stage(hq, hk, hv)
            self._chk(lib.tts_decode_step(h, 1, self.req, None, k.data_ptr(), v.data_ptr(), q.data_ptr(),
                                          self.scale, out.data_ptr(), st), "decode_step")
            if e2e is not None:
                e2e["pipe"].release()
            if stats_accum is not None:
                self._chk(lib.tts_block_table_stats(h, 1, self.req, None, stats_accum[self.ncall].data_ptr(), st),
                          "stats")
                self.ncall += 1
            if seg is not None and (it.forks or it is self.sched[-1]):
                e_end = torch.cuda.Event(enable_timing=True)
                e_end.record(torch.cuda.current_stream(self.dev))
                seg.append((open_ev, e_end))
                open_ev = None
            for (_, s) in it.forks:
                sc = self.scores[s]
                if self.world > 1:  # this rank's beams' scores, in its row order (ascending gid)
                    sc = sc[torch.tensor(self.ctx.tts_span_gids(0), device=self.dev)].contiguous()
                if e2e is not None:
                    sc = sc.cpu().pin_memory().to(self.dev, non_blocking=True)
                    e2e["h2d"] += sc.numel() * 4
                    e2e["d2h"] += c.N * 4
                if forks is not None:
                    f0 = torch.cuda.Event(enable_timing=True)
                    f0.record(torch.cuda.current_stream(self.dev))
                if self.world > 1:
                    self.ctx.tts_beam_select_fork_global(0, sc, c.M)
                else:
                    self.ctx.tts_beam_select_fork([0], sc.view(1, -1), c.M)
                if forks is not None:
                    f1 = torch.cuda.Event(enable_timing=True)
                    f1.record(torch.cuda.current_stream(self.dev))
                    forks.append((f0, f1))
        if e2e is not None:
            e2e["pipe"].drain()
        self._chk(lib.tts_block_table_release_request(h, 0, st), "release")


# ---------------------------------------------------------------------------
# CPU baseline: the fp64 oracle as it stands (oracle/run.py), on a bounded
# sample of the same workload (SURVEY 8(d) "Oracle beside it").
_ORC = {}


def _oracle_task(task):
    """Worker: one oracle attention call, OracleRun.beam_output, for a beam
    whose token-identity list is given (one layer).  Returns its duration."""
    cfg, r, b, t, l, ident = task
    torch.set_num_threads(1)
    from oracle.run import OracleRun
    orc = _ORC.get(cfg.name)
    if orc is None:
        orc = _ORC[cfg.name] = OracleRun(cfg.with_(R=r + 1), track_content=False)
        orc.lists = {}
    orc.lists[r] = {b: ident}
    t0 = time.perf_counter()
    orc.beam_output(r, b, t, l)
    return time.perf_counter() - t0


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "?"


def cpu_baseline(cfg, seconds, cores=None):
    """The oracle as it stands, timed on the host cores on a bounded sample:
    * the block-table simulator + per-beam identity lists over the schedule of
      request 0 (every append and EVERY fork, each fork timed; stopped and
      extrapolated per position if it exceeds a third of the budget);
    * fp64 attention (OracleRun.beam_output) at the first, middle and last
      position of every TTS step, on a spread subset of the active beams and
      one layer (all layers cost the same), run once on one core and once on
      all cores (a process pool, one thread per process); per-position cost is
      interpolated linearly within each step and multiplied by the active beams
      and L layers (the extrapolation factor is returned).
    beam-steps/s = beam-steps / (attention estimate + simulator time)."""
    import multiprocessing as mproc

    from oracle.run import OracleRun
    cores = cores or len(os.sched_getaffinity(0))
    c1 = cfg.with_(R=1)
    sched = list(workload.schedule(c1, [0]))
    orc = OracleRun(c1, track_content=False)
    orc.install()
    # --- pass 1: simulator (appends, forks) and the sample positions
    steps_pos = []          # per TTS step: its iterations
    cur = []
    for it in sched:
        cur.append(it.t)
        if it.forks or it is sched[-1]:
            steps_pos.append(cur)
            cur = []
    want = set()
    for pos in steps_pos:
        want.update({pos[0], pos[len(pos) // 2], pos[-1]})
    tasks, fork_s = [], []
    t_sim = 0.0
    done_pos = 0
    budget_sim = seconds / 3
    n_beam_sample = 4
    active_n = {}
    for it in sched:
        t0 = time.perf_counter()
        orc.sim.append(it.reqs, [a.tolist() for a in it.active], None)
        act = it.active[0]
        idx = np.nonzero(act)[0]
        for b in idx:
            orc.lists[0][b] = np.concatenate([orc.lists[0][b], [[it.t, b]]])
        t_sim += time.perf_counter() - t0
        active_n[it.t] = int(act.sum())
        done_pos += 1
        if it.t in want and len(idx):
            pick = idx[np.linspace(0, len(idx) - 1, min(n_beam_sample, len(idx))).astype(int)]
            for b in sorted(set(pick.tolist())):
                tasks.append((c1, 0, int(b), it.t, 0, orc.lists[0][b].copy()))
        if it.forks:
            t0 = time.perf_counter()
            sc = workload.scores(c1, 0, it.forks[0][1]).tolist()
            parents = orc.sim.fork([0], [sc], c1.M)[0]
            orc.lists[0] = [orc.lists[0][parents[c]].copy() for c in range(c1.N)]
            dt = time.perf_counter() - t0
            fork_s.append(dt)
            t_sim += dt
        if t_sim > budget_sim and it is not sched[-1]:
            break
    n_pos_total = len(sched)
    beam_steps_total = sum(int(it.active[0].sum()) for it in sched)
    sim_extrap = n_pos_total / done_pos
    t_sim_total = t_sim * sim_extrap
    # --- pass 2: attention samples, one core then all cores
    tasks = [tk for tk in tasks if tk[3] <= sched[done_pos - 1].t]
    ctx = mproc.get_context("spawn")
    with ctx.Pool(cores) as pool:
        pool.map(_oracle_task, tasks[:1] * cores, chunksize=1)   # warm every worker (imports, prompt K/V)
        per = pool.map(_oracle_task, [tasks[0], tasks[-1]])      # calibrate
        est = max(1e-4, sum(per) / 2)
        keep = max(cores, min(len(tasks), int(seconds / 3 / est * cores)))
        sel = sorted(set(np.linspace(0, len(tasks) - 1, keep).astype(int).tolist()))
        tasks = [tasks[i] for i in sel]
        w0 = time.perf_counter()
        pool.map(_oracle_task, tasks, chunksize=1)
        wallc = time.perf_counter() - w0
    # one core: an evenly spaced subset of the same calls (~ a third of the budget)
    keep1 = max(2, min(len(tasks), int(seconds / 3 / est)))
    tasks1 = [tasks[i] for i in sorted(set(np.linspace(0, len(tasks) - 1, keep1).astype(int).tolist()))]
    with ctx.Pool(1) as pool:
        pool.map(_oracle_task, tasks1[:1])
        w0 = time.perf_counter()
        dur1 = pool.map(_oracle_task, tasks1)
        wall1 = time.perf_counter() - w0
    speedup = max(1.0, (len(tasks) / wallc) / (len(tasks1) / wall1))
    # per-position single-core attention cost: mean over the position's sampled
    # beams x active beams x L, interpolated linearly between sampled positions
    per_pos = {}
    for tk, d in zip(tasks1, dur1):
        per_pos.setdefault(tk[3], []).append(d)
    xs = sorted(per_pos)
    ys = [float(np.mean(per_pos[x])) for x in xs]
    t_attn1 = 0.0
    for it in sched:
        t_attn1 += float(np.interp(it.t, xs, ys)) * active_n.get(it.t, int(it.active[0].sum())) * cfg.L
    value_1 = beam_steps_total / (t_attn1 + t_sim_total)
    value_c = beam_steps_total / (t_attn1 / speedup + t_sim_total)
    n_attn_calls = sum(int(it.active[0].sum()) for it in sched) * cfg.L
    return {"value": value_c, "unit": UNIT, "cores": cores, "kind": "oracle",
            "value_1core": value_1, "cores_1core": 1, "cpu_model": _cpu_model(),
            "host_cores": os.cpu_count(), "parallel_speedup": speedup,
            "fork_us_per_call": 1e6 * float(np.mean(fork_s)) if fork_s else None, "forks_timed": len(fork_s),
            "sample": (f"{cfg.name}, request 0: block-table simulator + identity lists over "
                       f"{done_pos}/{n_pos_total} positions (x{sim_extrap:.2f} extrapolated, {len(fork_s)} forks "
                       f"each timed, {t_sim:.1f} s); fp64 attention at the first/middle/last position of every "
                       f"TTS step on a spread subset of <= {n_beam_sample} active beams, layer 0: {len(tasks)} "
                       f"(beam, layer) calls on {cores} cores (process pool, {wallc:.1f} s), {len(tasks1)} of them "
                       f"on 1 core ({wall1:.1f} s); the run has {n_attn_calls} such calls "
                       f"(extrapolation x{n_attn_calls / max(1, len(tasks1)):.0f}, linear in position within a step)")}


def run_reference(args):
    ws, rank, local = dist_init(args.gpus)
    if rank != 0:
        return
    cfg = workload.CONFIGS[resolve_config(args, ws)]
    t0 = time.perf_counter()
    vals = []
    # each step a bounded sample; the whole K + W run stays within a few minutes
    per = min(args.cpu_seconds, max(3.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        cpu_baseline(cfg, min(per, 3.0))
    for _ in range(args.steps):
        vals.append(cpu_baseline(cfg, per))
    v = statistics.median([x["value"] for x in vals])
    cb = dict(vals[-1])
    cb["value"] = v
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "parallelism": "cpu oracle (rank 0 only)"},
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": time.perf_counter() - t0}
    print(json.dumps(line))


def position_bound(per_call, cfg, read_gbs, tc_flops, mufu_per_s):
    """per decode call (one position of the call's requests, all
    layers) the time bound max(U / BW, F / TC, E / MUFU) -- U unique KV bytes
    (+ q, out), F = 4 d Hq L x (sum of active lengths) FLOPs of QK^T and PV, E =
    Hq L x (sum of active lengths) exponentials.  Returns (sum of bounds in s,
    the fraction of calls each resource bounds)."""
    u = per_call[:, 0].astype(np.float64)
    lg = per_call[:, 1].astype(np.float64)
    kv_tok = 4 * cfg.Hkv * cfg.d * cfg.L
    t_mem = u * kv_tok / (read_gbs * 1e9)
    t_mma = 4.0 * cfg.d * cfg.Hq * cfg.L * lg / tc_flops
    t_exp = cfg.Hq * cfg.L * lg / mufu_per_s
    tb = np.maximum(np.maximum(t_mem, t_mma), t_exp)
    n = max(1, len(tb))
    which = {"hbm": float((t_mem >= np.maximum(t_mma, t_exp)).sum() / n),
             "tensor": float((t_mma > np.maximum(t_mem, t_exp)).sum() / n),
             "mufu": float((t_exp > np.maximum(t_mem, t_mma)).sum() / n)}
    return float(tb.sum()), which


def main():
    args = parse()
    maybe_spawn(args)
    if args.impl == "reference":
        return run_reference(args)
    ws, rank, local = dist_init(args.gpus)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cname = resolve_config(args, ws)
    cfg = workload.CONFIGS[cname]
    rot = args.rotate or DEFAULT_ROTATE[cname]
    if args.tts_steps:
        cfg = cfg.with_(n_steps=args.tts_steps)
    ppr = args.pages_per_request
    span = cname == "C5"
    if span:
        # one request, its N beams spread over the ranks; global top-K each step
        scaling = "strong"
        b = SpanBench(cfg, ws, rank, local)
        greqs = [0]
    elif cfg.step_len == 0:
        # straggler batch: shard the R requests over ranks (request r -> rank r mod G).
        # The 64-request batch is defined for 2/4/8 GPUs; its page pool does not
        # fit one GPU (64 x 6000 pages x 459 KB), so N = 1 runs the 4-GPU shard
        # (16 requests) unless --requests says otherwise.
        if args.requests:
            cfg = cfg.with_(R=args.requests)
        elif ws == 1:
            cfg = cfg.with_(R=16)
        greqs = [r for r in range(cfg.R) if r % ws == rank]
        scaling = "strong"
    else:
        cfg = cfg.with_(R=rot * ws)  # independent requests of the same shape, rot per rank
        greqs = [rank * rot + i for i in range(rot)]
        scaling = "weak"
    if not span:
        b = Bench(cfg, greqs, local, pages_per_request=ppr, per_call=args.per_call or DEFAULT_PER_CALL[cname])
    st = torch.cuda.current_stream(dev)

    # read-only HBM stream peak of this device (the attention
    # kernel's read roofline, beside the copy peak of MEASURED_PEAKS.json)
    from paper_2509_00195_b200 import tts as tts_mod
    probe = torch.empty(4 << 30, dtype=torch.uint8, device=dev)
    probe.fill_(1)
    read_gbs = max(tts_mod.stream_read_gbs(probe, 10) for _ in range(3))
    del probe
    torch.cuda.empty_cache()

    # warm-up (the first one also accumulates the unique / logical KV statistics)
    per_call = torch.zeros(b.n_calls, 2, dtype=torch.int64, device=dev)  # unique / logical tokens per call
    for i in range(max(args.warmup, 1)):
        b.run_step(stats_accum=per_call if i == 0 else None)
    torch.cuda.synchronize(dev)
    st_code = b.ctx.tts_device_status()
    assert st_code == 0, f"device status {st_code} during warm-up"
    per_call_np = per_call.cpu().numpy()
    unique_tok, logical_tok = [int(x) for x in per_call_np.sum(0).tolist()]
    kv_tok = 4 * cfg.Hkv * cfg.d * cfg.L  # bytes per token over all layers (bf16 K+V)
    if args.dump_call_bytes:
        # algorithmic bytes of every attention launch of one step (to line up with ncu launch ids)
        active_rows = [int(a.sum()) for it in b.sched for a in (it.active if not b.batched else [np.stack(it.active)])]
        calls = per_call_np[:, 0].tolist()
        json.dump({"config": cfg.name, "kv_bytes_per_token": kv_tok,
                   "qo_bytes_per_beam": cfg.L * cfg.Hq * cfg.d * 6,
                   "unique_kv_bytes": [u * kv_tok for u in calls], "active_beams": active_rows},
                  open(args.dump_call_bytes, "w"))
    unique_b, logical_b = unique_tok * kv_tok, logical_tok * kv_tok
    qo_b = b.beam_steps * cfg.L * cfg.Hq * cfg.d * (2 + 4)

    # timed region (no per-launch instrumentation: the headline value)
    clocks = Clocks(local)
    launches0 = b.ctx.launch_count()
    barrier(ws)
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    h0 = time.perf_counter()
    for _ in range(args.steps):
        b.run_step()
    host_s = time.perf_counter() - h0  # host enqueue time (the GPU may still be running)
    e1.record(st)
    torch.cuda.synchronize(dev)
    barrier(ws)
    ms = e0.elapsed_time(e1)
    launches = b.ctx.launch_count() - launches0
    clk = clocks.stop()
    assert b.ctx.tts_device_status() == 0, "device status error in timed region"

    # kernel-duration pass: the same K steps again, with a CUDA event pair on the
    # launching stream around every run of decode calls between two forks (the
    # decode-step kernels: k_plan + k_tree_umma per call, k_alloc on page
    # crossings) and around every select + fork.  Events between individual
    # calls would serialise the programmatic-dependent-launch overlap of
    # consecutive calls, so they are only placed where a fork breaks it anyway.
    segs, fks = [], []
    barrier(ws)
    torch.cuda.synchronize(dev)
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record(st)
    for _ in range(args.steps):
        b.run_step(seg=segs, forks=fks)
    p1.record(st)
    torch.cuda.synchronize(dev)
    barrier(ws)
    ms_prof = p0.elapsed_time(p1)
    attn_ms = sum(a.elapsed_time(z) for a, z in segs)
    fork_us = [a.elapsed_time(z) * 1e3 for a, z in fks]
    attn_launches = b.n_calls * args.steps
    assert b.ctx.tts_device_status() == 0, "device status error in profiled pass"

    ms_max = allmax(ms, ws, dev)
    total_steps = allsum(b.beam_steps * args.steps, ws, dev)
    value = total_steps / (ms_max / 1e3)
    pk, pk_src = peaks()
    attn_s = attn_ms / 1e3
    achieved_gbs = (unique_b + qo_b) * args.steps / attn_s / 1e9
    unique_gbs = unique_b * args.steps / attn_s / 1e9
    logical_gbs = logical_b * args.steps / attn_s / 1e9
    pj = {}
    pkf = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pkf):
        pj = json.load(open(pkf))
    tc = float(pj.get("bf16_tflops_sustained", 1407.4)) * 1e12
    sm_mhz = (clk or {}).get("sm_mhz") or float(pj.get("sm_max_mhz", 1965.0))
    mufu = torch.cuda.get_device_properties(dev).multi_processor_count * 16 * sm_mhz * 1e6
    tb, tb_which = position_bound(per_call_np, cfg, read_gbs, tc, mufu)
    tb *= args.steps

    # e2e: the same metric through the C-ABI with host buffers (pinned): every
    # call's q/k/v H2D and its output D2H (overlapped with the kernels on two
    # copy streams), the fork scores H2D and the parent maps D2H
    e2e = None
    if args.e2e_steps > 0:
        ring = [(q.cpu().pin_memory(), k.cpu().pin_memory(), v.cpu().pin_memory()) for q, k, v in b.ring]
        q0, k0, v0 = b.ring[0]
        pipe = IOPipe((q0, k0, v0), b.out, dev)
        ctx_e = {"ring": ring, "pipe": pipe, "d2h": 0, "h2d": 0, "parents": []}
        n_in = sum(1 for it in b.sched for _ in (it.reqs if not b.batched else [0]))
        barrier(ws)
        torch.cuda.synchronize(dev)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(st)
        for _ in range(args.e2e_steps):
            b.run_step(e2e=ctx_e)
        t1.record(st)
        torch.cuda.synchronize(dev)
        ems = allmax(t0.elapsed_time(t1), ws, dev)
        h2d = n_in * (q0.numel() * 2 + k0.numel() * 2 + v0.numel() * 2) * args.e2e_steps + ctx_e["h2d"]
        d2h = pipe.d2h_bytes + ctx_e["d2h"]
        e2e = {"value": allsum(b.beam_steps * args.e2e_steps, ws, dev) / (ems / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d / args.e2e_steps), "d2h_bytes_per_step": int(d2h / args.e2e_steps),
               "note": ("through tts_decode_step / tts_beam_select_fork with host buffers: every call's q/k/v "
                        "copied H2D and its fp32 output D2H (pinned, two copy streams overlapping the kernels), "
                        "PRM scores H2D and parent maps D2H per fork; bound by PCIe, not by the kernels")}

    # DRAM traffic of one ncu --set full capture of this kernel on this workload
    # (profiles/ncu_traffic_<cfg>.json, written by tools/profile_summary.py),
    # scaled to this run's average launch by the captured launch's traffic /
    # algorithmic-bytes ratio (1.0 = every unique page read from HBM exactly once)
    traffic, traffic_algo, traffic_src = None, None, None
    prof = os.path.join(ROOT, "profiles", f"ncu_traffic_{cname}.json")
    if os.path.exists(prof):
        try:
            pjf = json.load(open(prof))
            traffic = float(pjf["dram_bytes_per_launch"])
            traffic_algo = float(pjf["algo_bytes_of_that_launch"])
            traffic_src = f"profiles/ncu_traffic_{cname}.json ({pjf.get('tag', '?')}: one --set full capture)"
        except Exception:
            traffic = None

    cb = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline(cfg, args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": cfg.name, "requests_per_rank": len(greqs), "N": cfg.N, "M": cfg.M,
                       "L": cfg.L, "Hq": cfg.Hq, "Hkv": cfg.Hkv, "d": cfg.d, "page": cfg.P,
                       "prompt": cfg.prompt, "steps_x_len": f"{cfg.n_steps}x{cfg.step_len or 'lognormal'}",
                       "beam_steps_per_rank_step": b.beam_steps,
                       "l2": (f"unique KV per call {unique_b / max(1, b.n_calls) / 1e6:.0f} MB vs 126 MB L2; "
                              + ("one request whose beams span the ranks" if span else
                                 f"rotation over {len(greqs)} independent requests, {b.per_call} per call"
                                 if not b.batched else "batched requests")),
                       "parallelism": (f"beam-sharded x{ws} (one request's beams span the ranks; NCCL all-gather "
                                       "of scores + lineage migration per step)" if span else
                                       f"dp{ws} (independent requests per rank, no data-path collective)")},
            "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": pk, "unit": "GB/s",
                         "frac": achieved_gbs / pk, "traffic": traffic,
                         "traffic_algo_bytes_of_captured_launch": traffic_algo,
                         "traffic_over_algo": (traffic / traffic_algo) if traffic and traffic_algo else None,
                         "traffic_source": traffic_src,
                         "peak_source": pk_src,
                         "kernel": "decode step: k_plan (a2 append + a3 plan) + k_tree_umma (a4/a5 tcgen05 "
                                   "prefix-shared attention), PDL-chained; + k_alloc on page crossings",
                         "algo_bytes": "unique KV (valid tokens of distinct pages) + q bf16 + out fp32",
                         "algo_bytes_per_launch": (unique_b + qo_b) / max(1, b.n_calls),
                         "read_peak_gbs_measured": read_gbs,
                         "frac_of_read_peak": achieved_gbs / read_gbs,
                         "unique_kv_gbs": unique_gbs, "unique_kv_frac_of_8tbs": unique_gbs / HBM_SPEC_GBS,
                         "unique_kv_frac_of_read_peak": unique_gbs / read_gbs,
                         "logical_kv_gbs": logical_gbs, "reuse": logical_tok / max(unique_tok, 1),
                         "position_bound_ms_per_step": tb * 1e3 / args.steps,
                         "frac_of_position_bound": tb / attn_s,
                         "position_bound_by": tb_which,
                         "position_bound_rates": {"read_gbs": read_gbs, "tensor_tflops": tc / 1e12,
                                                  "mufu_ex2_per_s": mufu},
                         "attn_ms_per_step": attn_ms / args.steps, "attn_launches_per_step": attn_launches // args.steps,
                         "attn_us_per_launch": attn_ms * 1e3 / max(attn_launches, 1),
                         "attn_share_of_step": attn_ms / ms_prof,
                         "timing": "separate K-step pass, a CUDA event pair on the launching stream around every "
                                   f"run of decode calls between forks ({len(segs)} pairs; "
                                   f"{ms_prof / args.steps:.1f} ms/step with events vs {ms / args.steps:.1f} clean)"},
            "select_fork_us_per_call": float(np.mean(fork_us)) if fork_us else None,
            "select_fork_calls_per_step": len(fork_us) // max(1, args.steps),
            "cpu_baseline": cb,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "attention_kernel": b.ctx.attention_kernel(),
            "host_enqueue_ms_per_step": host_s * 1e3 / args.steps,
            "clocks": clk,
        }
        print(json.dumps(line))
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
