"""Speculative Beam Extension (f1) on a straggler-heavy C4-shaped workload,
speculation off vs on, same inputs: slot occupancy (rows generating / slots),
decode iterations, non-speculative beam-steps, speculative tokens, head-start
tokens kept, and device time (CUDA events; the loop's host bookkeeping runs
between calls).  usage: python tools/spec_bench.py [R] [N] [steps] [L]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_00195_b200 import build  # noqa: E402

build.build()
from paper_2509_00195_b200.runner import SpecBeamRunner  # noqa: E402
from synth import workload  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 2
N = int(sys.argv[2]) if len(sys.argv) > 2 else 64
S = int(sys.argv[3]) if len(sys.argv) > 3 else 4
L = int(sys.argv[4]) if len(sys.argv) > 4 else 28
cfg = workload.C4.with_(R=R, N=N, n_steps=S, L=L)
out = {"workload": f"{cfg.name} R={R} N={N} M={cfg.M} steps={S} L={L} (log-normal step lengths)"}
for spec in (False, True):
    run = SpecBeamRunner(cfg, spec=spec)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    st = run.run()
    e1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    assert run.ctx.tts_device_status() == 0
    out["on" if spec else "off"] = {
        "occupancy": sum(st["running"]) / sum(st["capacity"]), "iterations": st["iterations"],
        "beam_steps": st["beam_steps"], "spec_tokens": st["spec_tokens"],
        "device_ms": e0.elapsed_time(e1), "wall_s": wall,
        "beam_steps_per_s_wall": st["beam_steps"] / wall}
print(json.dumps(out))
