"""Build libtts with -DTTS_TRACE and run a config through BeamStepRunner; print
per-call timelines from the launch spans (globaltimer): attention kernel span
(first CTA start -> last CTA exit), k_plan span, and the gap between one
call's last attention exit and the next call's first attention start.
usage: python tools/spans.py <config> [tts_steps]"""
import ctypes
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2509_00195_b200 import build  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 0
lib = build.LIB.replace("libtts.so", "libtts_trace.so")
cmd = [build.NVCC, *build.ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC", "-DTTS_TRACE",
       *sys.argv[3:], "-I", os.path.join(build.ROOT, "include"), "-o", lib, *build.sources()]
subprocess.run(cmd, check=True, capture_output=True)
from paper_2509_00195_b200 import tts  # noqa: E402

tts.LIB_PATH = lib
import torch  # noqa: E402

from paper_2509_00195_b200.runner import BeamStepRunner  # noqa: E402
from synth import workload  # noqa: E402

cfg = workload.CONFIGS[name]
if steps:
    cfg = cfg.with_(n_steps=steps)
r = BeamStepRunner(cfg)
L = tts.load()
torch.cuda.synchronize()
L.tts_debug_reset_spans()
r.run()
torch.cuda.synchronize()
buf = np.zeros((32768, 4), dtype=np.uint64)
L.tts_debug_read_spans(buf.ctypes.data_as(ctypes.c_void_p))
ok = (buf[:, 1] > 0) & (buf[:, 0] < np.uint64(2 ** 63))
b = buf[ok].astype(np.float64)
b = b[np.argsort(b[:, 0])]
t0 = b[0, 0]
att = (b[:, 1] - b[:, 0]) / 1e3
plan = np.where(b[:, 3] > 0, (b[:, 3] - b[:, 2]) / 1e3, np.nan)
gap = (b[1:, 0] - b[:-1, 1]) / 1e3
period = (b[1:, 0] - b[:-1, 0]) / 1e3
print(f"{name}: {len(b)} attention launches; total {(b[-1, 1] - t0) / 1e6:.1f} ms")
for nm, x in (("attention span us", att), ("k_plan span us", plan), ("gap exit->next start us", gap),
              ("start->next start us", period)):
    x = x[np.isfinite(x)]
    print(f"  {nm:26s} mean {x.mean():8.2f}  p10 {np.percentile(x, 10):8.2f}  p50 {np.median(x):8.2f}  "
          f"p90 {np.percentile(x, 90):8.2f}  max {x.max():8.2f}  sum {x.sum() / 1e3:9.1f} ms")
big = np.argsort(gap)[-8:]
print("  largest gaps (launch idx, us):", [(int(i), round(float(gap[i]), 1)) for i in big])
# plan start relative to the previous attention exit
ps = (b[1:, 2] - b[:-1, 1]) / 1e3
pe = (b[1:, 3] - b[:-1, 1]) / 1e3
print(f"  k_plan start - prev attn exit: p50 {np.median(ps):.2f} us; k_plan end - prev attn exit: p50 {np.median(pe):.2f} us")
n = len(b)
for frac in (0.1, 0.5, 0.9):
    i = int(frac * (n - 1))
    print(f"  launch {i}: attn {att[i]:.1f} us, gap after {gap[min(i, n - 2)]:.2f} us")
