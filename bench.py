#!/usr/bin/env python
"""Benchmark of the FlashTTS beam-step hot path on B200 (libtts through its C-ABI).

One bench *step* = one complete TTS run of the configuration for every
request a rank holds: install on the prompt, every decode iteration (append +
prefix-shared attention over all L layers), a select + fork after every TTS
step but the last, release.  All SURVEY 8(a) rows are inside the timed region.

Workload (BASELINE.json configs): default C2 (configs[1], Qwen2.5-Math-1.5B
attention shape, N=16, M=4, 2k-token chains).  L2 control: each rank rotates
--rotate independent requests of that shape, one request per C-ABI call, so
the reuse distance of any KV page between two positions is >= 2x the 126 MB
L2 (SURVEY 8(d) pitfall 1: "rotate across independent request pools").
Multi-GPU: one process per GPU, each with its own requests (no collective on
the data path; SURVEY 8(e) C4 partitioning) -> "scaling": "weak".

--impl reference times the CPU oracle (the only reference this paper-only
task has) on the host cores, on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
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
DEFAULT_ROTATE = {"C1": 64, "C2": 32, "C3": 4, "C4": 1, "C5": 1}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="libtts", choices=["libtts", "reference"])
    ap.add_argument("--config", default="C2", choices=list(workload.CONFIGS))
    ap.add_argument("--rotate", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--dump-call-bytes", default="")
    ap.add_argument("--requests", type=int, default=0, help="override R of the straggler batch (C4)")
    ap.add_argument("--tts-steps", type=int, default=0, help="override the number of TTS steps (shorter chains)")
    ap.add_argument("--pages-per-request", type=int, default=0,
                    help="page-pool budget per request (default: exact bound for fixed steps, 6000 for C4)")
    return ap.parse_args()


def dist_init(n):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
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
class H2DPipe:
    """Double-buffered host -> device staging of each call's inputs on a copy
    stream, so that the next call's q/k/v copy overlaps this call's kernels
    (the way a serving loop feeds the C-ABI from pinned host memory)."""

    def __init__(self, like, dev):
        self.slots = [tuple(torch.empty_like(t) for t in like) for _ in range(2)]
        self.cs = torch.cuda.Stream(dev)
        self.ready = [torch.cuda.Event() for _ in range(2)]
        self.free = [torch.cuda.Event() for _ in range(2)]
        self.i = 0
        self.dev = dev

    def stage(self, hq, hk, hv):
        s = self.i & 1
        with torch.cuda.stream(self.cs):
            self.cs.wait_event(self.free[s])  # the call that last used this slot has run
            q, k, v = self.slots[s]
            q.copy_(hq, non_blocking=True)
            k.copy_(hk, non_blocking=True)
            v.copy_(hv, non_blocking=True)
            self.ready[s].record(self.cs)
        torch.cuda.current_stream(self.dev).wait_event(self.ready[s])
        return q, k, v

    def release(self):
        self.free[self.i & 1].record(torch.cuda.current_stream(self.dev))
        self.i += 1


# ---------------------------------------------------------------------------
class Bench:
    """Drives one rank's requests through libtts with minimal host overhead."""

    def __init__(self, cfg, greqs, dev_index, ring=8, pages_per_request=0):
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
        per_call = self.n if self.batched else 1
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
        self.parent = torch.empty(self.n, cfg.N, dtype=torch.int32, device=self.dev)
        self.beam_steps = sum(int(a.sum()) for it in self.sched for a in it.active)
        self.stream = self.ctx.stream
        self.ncall = 0
        self.n_calls = sum(1 if self.batched else len(it.reqs) for it in self.sched)
        torch.cuda.synchronize(self.dev)

    def _chk(self, code, what):
        if code != 0:
            from paper_2509_00195_b200.tts import TTSError
            raise TTSError(code, what)

    def run_step(self, stats_accum=None, e2e=None, seg=None):
        """One full run of every request.  e2e: dict of pinned host rings to copy from.
        seg: list receiving one CUDA event pair (on the launching stream) per run of
        consecutive decode calls between two forks (install / release excluded)."""
        c = self.cfg
        open_ev = None
        lib, h, st = self.lib, self.h, self.stream
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
            if seg is not None and open_ev is None:
                open_ev = torch.cuda.Event(enable_timing=True)
                open_ev.record(torch.cuda.current_stream(self.dev))
            if e2e is None and not self.batched and stats_accum is None:
                # hot loop: one C-ABI call per request and position, arguments pre-marshalled
                qp, kp, vp = ptrs[it.t % nr]
                for r in it.reqs:
                    rc = decode(h, 1, self.req_arr[self.local[r]], None, kp, vp, qp, self.scale, outp, st)
                    if rc:
                        self._chk(rc, "decode_step")
            else:
                if e2e is not None:
                    hq, hk, hv = e2e["ring"][it.t % nr]
                if self.batched:
                    if e2e is not None:
                        q, k, v = e2e["pipe"].stage(hq, hk, hv)
                    loc = [self.local[r] for r in it.reqs]
                    arr = (ctypes.c_int32 * len(loc))(*loc)
                    act = np.ascontiguousarray(np.stack(it.active), dtype=np.uint8)
                    self._chk(lib.tts_decode_step(h, len(loc), arr, act.ctypes.data_as(ctypes.c_void_p),
                                                  k.data_ptr(), v.data_ptr(), q.data_ptr(), self.scale,
                                                  self.out.data_ptr(), st), "decode_step")
                    if e2e is not None:
                        e2e["pipe"].release()
                    if stats_accum is not None:
                        self._chk(lib.tts_block_table_stats(h, len(loc), arr, act.ctypes.data_as(ctypes.c_void_p),
                                                            stats_accum[self.ncall].data_ptr(), st), "stats")
                        self.ncall += 1
                else:
                    for ri, r in enumerate(it.reqs):
                        if e2e is not None:  # every call's q/k/v come from the host
                            q, k, v = e2e["pipe"].stage(hq, hk, hv)
                        arr = self.req_arr[self.local[r]]
                        self._chk(lib.tts_decode_step(h, 1, arr, None, k.data_ptr(), v.data_ptr(), q.data_ptr(),
                                                      self.scale, self.out.data_ptr(), st), "decode_step")
                        if e2e is not None:
                            e2e["pipe"].release()
                        if stats_accum is not None:
                            self._chk(lib.tts_block_table_stats(h, 1, arr, None, stats_accum[self.ncall].data_ptr(),
                                                                st), "stats")
                            self.ncall += 1
            if it.forks or (seg is not None and it is self.sched[-1]):
                if seg is not None:
                    e_end = torch.cuda.Event(enable_timing=True)
                    e_end.record(torch.cuda.current_stream(self.dev))
                    seg.append((open_ev, e_end))
                    open_ev = None
            if it.forks:
                loc = [self.local[r] for r, _ in it.forks]
                arr = (ctypes.c_int32 * len(loc))(*loc)
                sc = torch.stack([self.scores[(r, s)] for r, s in it.forks]) if len(loc) > 1 else \
                    self.scores[it.forks[0]].view(1, -1)
                if e2e is not None:
                    sc = sc.cpu().pin_memory().to(self.dev, non_blocking=True)
                self._chk(lib.tts_beam_select_fork(h, len(loc), arr, sc.data_ptr(), c.M,
                                                   self.parent.data_ptr(), st), "select_fork")
                if e2e is not None:
                    e2e["d2h"] += self.parent[: len(loc)].numel() * 4
                    e2e["parents"].append(self.parent[: len(loc)].to("cpu", non_blocking=True))
        if e2e is not None:
            e2e["last_out"].copy_(self.out, non_blocking=True)
            e2e["d2h"] += self.out.numel() * 4
        for r in self.greqs:
            self._chk(lib.tts_block_table_release_request(h, self.local[r], st), "release")


class SpanBench:
    """C5: one request whose N beams span the G ranks (n = N / G per rank).
    Per decode iteration each rank runs append + attention on its n beams;
    at every step end the ranks all-gather scores and lengths (NCCL), run the
    same global selection and migrate lineages whose children changed rank
    (paper_2509_00195_b200.dist.select_fork_global)."""

    def __init__(self, cfg, world, rank, dev_index, ring=8):
        from paper_2509_00195_b200 import build
        build.build()
        from paper_2509_00195_b200.runner import tts_config, Inputs
        from paper_2509_00195_b200.tts import Context
        self.cfg, self.world, self.rank = cfg, world, rank
        self.nl = cfg.N // world
        maxb = 2 * self.nl if world > 1 else cfg.N
        from paper_2509_00195_b200.runner import pages_per_request
        if world == 1:
            pages = pages_per_request(cfg) + 256  # the whole tree on one rank
        else:
            pages = self.nl * workload.max_pages_per_beam(cfg) + 256  # imported lineages are private copies
        self.tcfg = tts_config(cfg, 1, num_pages=pages, max_beams=maxb)
        self.ctx = Context(self.tcfg, dev_index)
        self.lib, self.h, self.dev = self.ctx.lib, self.ctx.h, self.ctx.device
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
        sl = slice(rank * self.nl, (rank + 1) * self.nl)
        self.scores = {s: self.inp.scores(0, s)[sl].contiguous() for it in self.sched for (_, s) in it.forks}
        self.act = {}
        self.beam_steps = sum(int(it.active[0][sl].sum()) for it in self.sched)
        self.n_calls = len(self.sched)
        self.ncall = 0
        self.stream = self.ctx.stream
        self.req = (ctypes.c_int32 * 1)(0)
        torch.cuda.synchronize(self.dev)

    def _chk(self, code, what):
        if code != 0:
            from paper_2509_00195_b200.tts import TTSError
            raise TTSError(code, what)

    def run_step(self, stats_accum=None, e2e=None, seg=None):
        from paper_2509_00195_b200.dist import select_fork_global
        c, lib, h, st = self.cfg, self.lib, self.h, self.stream
        k, v = self.prompt
        self._chk(lib.tts_block_table_init_request(h, 0, self.nl, c.prompt, k.data_ptr(), v.data_ptr(), st), "init")
        nr = len(self.ring)
        open_ev = None
        for it in self.sched:
            q, k, v = self.ring[it.t % nr]
            if seg is not None and open_ev is None:
                open_ev = torch.cuda.Event(enable_timing=True)
                open_ev.record(torch.cuda.current_stream(self.dev))
            if e2e is not None:
                hq, hk, hv = e2e["ring"][it.t % nr]
                q, k, v = e2e["pipe"].stage(hq, hk, hv)
            self._chk(lib.tts_decode_step(h, 1, self.req, None, k.data_ptr(), v.data_ptr(), q.data_ptr(),
                                          self.scale, self.out.data_ptr(), st), "decode_step")
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
                if e2e is not None:
                    sc = sc.cpu().pin_memory().to(self.dev, non_blocking=True)
                    e2e["d2h"] += c.N * 4
                if self.world > 1:
                    select_fork_global(self.ctx, 0, sc, c.M)
                else:
                    self.ctx.tts_beam_select_fork([0], sc.view(1, -1), c.M)
        if e2e is not None:
            e2e["last_out"].copy_(self.out, non_blocking=True)
            e2e["d2h"] += self.out.numel() * 4
        self._chk(lib.tts_block_table_release_request(h, 0, st), "release")


def cpu_baseline(cfg, seconds):
    """The oracle as it stands, on a bounded sample: the first decode iterations
    of request 0 with full attention (all active beams x all layers) per
    iteration, until ~`seconds` of CPU work."""
    from oracle.run import OracleRun
    torch.set_num_threads(os.cpu_count() or 1)
    orc = OracleRun(cfg.with_(R=1), num_pages=None, track_content=False)
    t0 = time.perf_counter()
    n_iters = 0
    steps = 0
    state = {"stop": False}

    def sample(it):
        nonlocal n_iters, steps
        if state["stop"]:
            return []
        n_iters += 1
        pts = [(r, b, l) for k, r in enumerate(it.reqs) for b in range(cfg.N) if it.active[k][b]
               for l in range(cfg.L)]
        steps += len(pts) // cfg.L
        return pts

    class Stop(Exception):
        pass

    it_count = 0
    try:
        orc.install()
        for it in workload.schedule(cfg.with_(R=1), [0]):
            orc.sim.append(it.reqs, [a.tolist() for a in it.active], None)
            for k, r in enumerate(it.reqs):
                for b in np.nonzero(it.active[k])[0]:
                    orc.lists[r][b] = np.concatenate([orc.lists[r][b], [[it.t, b]]])
            for (r, b, l) in sample(it):
                orc.beam_output(r, b, it.t, l)
            it_count += 1
            if time.perf_counter() - t0 > seconds:
                break
    except Stop:
        pass
    dt = time.perf_counter() - t0
    return {"value": steps / dt, "unit": UNIT, "cores": torch.get_num_threads(), "kind": "oracle",
            "sample": f"{cfg.name}: first {it_count} decode iterations of one request, fp64 attention for "
                      f"all {cfg.N} beams x {cfg.L} layers per iteration ({steps} beam-steps, {dt:.1f} s)"}


def run_reference(args):
    ws, rank, local = dist_init(args.gpus)
    if rank != 0:
        return
    cfg = workload.CONFIGS[args.config]
    t0 = time.perf_counter()
    vals = []
    for _ in range(args.warmup):
        cpu_baseline(cfg, min(args.cpu_seconds, 5.0))
    for _ in range(args.steps):
        vals.append(cpu_baseline(cfg, args.cpu_seconds / max(args.steps, 1)))
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


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    ws, rank, local = dist_init(args.gpus)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = workload.CONFIGS[args.config]
    rot = args.rotate or DEFAULT_ROTATE[args.config]
    if args.tts_steps:
        cfg = cfg.with_(n_steps=args.tts_steps)
    ppr = args.pages_per_request
    span = args.config == "C5"
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
        # page budget: runner.pages_per_request (override with --pages-per-request)
    else:
        cfg = cfg.with_(R=rot * ws)  # independent requests of the same shape, rot per rank
        greqs = [rank * rot + i for i in range(rot)]
        scaling = "weak"
    if not span:
        b = Bench(cfg, greqs, local, pages_per_request=ppr)
    st = torch.cuda.current_stream(dev)

    # warm-up (the first one also accumulates the unique / logical KV statistics)
    per_call = torch.zeros(b.n_calls, 2, dtype=torch.int64, device=dev)  # unique / logical tokens per call
    for i in range(max(args.warmup, 1)):
        b.run_step(stats_accum=per_call if i == 0 else None)
    torch.cuda.synchronize(dev)
    st_code = b.ctx.tts_device_status()
    assert st_code == 0, f"device status {st_code} during warm-up"
    unique_tok, logical_tok = [int(x) for x in per_call.sum(0).tolist()]
    kv_tok = 4 * cfg.Hkv * cfg.d * cfg.L  # bytes per token over all layers (bf16 K+V)
    if args.dump_call_bytes:
        # algorithmic bytes of every attention launch of one step (to line up with ncu launch ids)
        active_rows = [int(a.sum()) for it in b.sched for a in (it.active if not b.batched else [np.stack(it.active)])]
        calls = per_call[:, 0].tolist()
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
    # crossings).  Events between individual calls would serialise the
    # programmatic-dependent-launch overlap of consecutive calls, so they are
    # only placed where a fork breaks the chain anyway.
    segs = []
    barrier(ws)
    torch.cuda.synchronize(dev)
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record(st)
    for _ in range(args.steps):
        b.run_step(seg=segs)
    p1.record(st)
    torch.cuda.synchronize(dev)
    barrier(ws)
    ms_prof = p0.elapsed_time(p1)
    attn_ms = sum(a.elapsed_time(z) for a, z in segs)
    attn_launches = b.n_calls * args.steps
    assert b.ctx.tts_device_status() == 0, "device status error in profiled pass"

    ms_max = allmax(ms, ws, dev)
    total_steps = allsum(b.beam_steps * args.steps, ws, dev)
    value = total_steps / (ms_max / 1e3)
    pk, pk_src = peaks()
    achieved_gbs = (unique_b + qo_b) * args.steps / (attn_ms / 1e3) / 1e9
    unique_gbs = unique_b * args.steps / (attn_ms / 1e3) / 1e9
    logical_gbs = logical_b * args.steps / (attn_ms / 1e3) / 1e9

    # e2e: same metric through the C-ABI with host buffers (pinned), H2D of every
    # iteration's q/k/v and the fork scores, D2H of the parent maps and the final output
    e2e = None
    if args.e2e_steps > 0:
        ring = [(q.cpu().pin_memory(), k.cpu().pin_memory(), v.cpu().pin_memory()) for q, k, v in b.ring]
        q0, k0, v0 = b.ring[0]
        ctx_e = {"ring": ring, "pipe": H2DPipe((q0, k0, v0), dev),
                 "d2h": 0, "parents": [], "last_out": torch.empty(b.out.shape, dtype=torch.float32).pin_memory()}
        h2d = sum(1 for it in b.sched for _ in (it.reqs if not b.batched else [0])) * \
            (q0.numel() * 2 + k0.numel() * 2 + v0.numel() * 2)
        h2d += sum(len(it.forks) for it in b.sched) * cfg.N * 4
        barrier(ws)
        torch.cuda.synchronize(dev)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(st)
        for _ in range(args.e2e_steps):
            ctx_e["d2h"] = 0
            b.run_step(e2e=ctx_e)
        t1.record(st)
        torch.cuda.synchronize(dev)
        ems = allmax(t0.elapsed_time(t1), ws, dev)
        e2e = {"value": allsum(b.beam_steps * args.e2e_steps, ws, dev) / (ems / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(ctx_e["d2h"])}

    # DRAM traffic of one ncu --set full capture of this kernel on this workload
    # (profiles/ncu_traffic_<cfg>.json, written by tools/profile_summary.py),
    # scaled to this run's average launch by the captured launch's traffic /
    # algorithmic-bytes ratio (1.0 = every unique page read from HBM exactly once)
    traffic, traffic_ratio = None, None
    prof = os.path.join(ROOT, "profiles", f"ncu_traffic_{args.config}.json")
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            traffic_ratio = pj["dram_bytes_per_launch"] / pj["algo_bytes_of_that_launch"]
            traffic = traffic_ratio * (unique_b + qo_b) / max(1, b.n_calls)
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
                       "l2": (f"rotation over {len(greqs)} independent requests, one per call" if not b.batched
                              else "batched requests (working set >> L2)"),
                       "parallelism": (f"beam-sharded x{ws} (one request's beams span the ranks; NCCL all-gather "
                                       "of scores + lineage migration per step)" if span else
                                       f"dp{ws} (independent requests per rank, no data-path collective)")},
            "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": pk, "unit": "GB/s",
                         "frac": achieved_gbs / pk, "traffic": traffic, "traffic_over_algo": traffic_ratio,
                         "peak_source": pk_src,
                         "kernel": "decode step: k_plan (a2 append + a3 plan) + k_tree_umma (a4/a5 tcgen05 "
                                   "prefix-shared attention), PDL-chained; + k_alloc on page crossings",
                         "algo_bytes": "unique KV (valid tokens of distinct pages) + q bf16 + out fp32",
                         "unique_kv_gbs": unique_gbs, "logical_kv_gbs": logical_gbs,
                         "reuse": logical_tok / max(unique_tok, 1),
                         "attn_ms_per_step": attn_ms / args.steps, "attn_launches_per_step": attn_launches // args.steps,
                         "attn_us_per_launch": attn_ms * 1e3 / max(attn_launches, 1),
                         "attn_share_of_step": attn_ms / ms_prof,
                         "timing": "separate K-step pass, a CUDA event pair on the launching stream around every "
                                   f"run of decode calls between forks ({len(segs)} pairs; "
                                   f"{ms_prof / args.steps:.1f} ms/step with events vs {ms / args.steps:.1f} clean)"},
            "cpu_baseline": cb,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "host_enqueue_ms_per_step": host_s * 1e3 / args.steps,
            "clocks": clk,
        }
        print(json.dumps(line))
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
