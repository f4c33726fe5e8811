"""Launch spans under bench.py's own hot loop (libtts built with -DTTS_TRACE):
per decode call, the attention kernel's span (first CTA start -> last CTA
exit), the gap to the next call's first CTA, and k_plan's span; the sum of
spans vs the step's wall time on the device.
usage: python tools/spans_bench.py <config> [per_call]"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2509_00195_b200 import build  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
per_call = int(sys.argv[2]) if len(sys.argv) > 2 else 1
lib = build.LIB.replace("libtts.so", "libtts_trace.so")
cmd = [build.NVCC, *build.ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC", "-DTTS_TRACE",
       "-I", os.path.join(ROOT, "include"), "-o", lib, *build.sources()]
subprocess.run(cmd, check=True, capture_output=True)
build.build()
from paper_2509_00195_b200 import tts  # noqa: E402

tts.LIB_PATH = lib
import torch  # noqa: E402

import bench  # noqa: E402
from synth import workload  # noqa: E402

cfg = workload.CONFIGS[name]
b = bench.Bench(cfg, list(range(cfg.R if name != "C4" else 16)), 0, per_call=per_call)
L = b.lib
b.run_step()
torch.cuda.synchronize()
L.tts_debug_reset_spans()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
b.run_step()
e1.record()
torch.cuda.synchronize()
step_ms = e0.elapsed_time(e1)
buf = np.zeros((32768, 4), dtype=np.uint64)
L.tts_debug_read_spans(buf.ctypes.data_as(ctypes.c_void_p))
ok = (buf[:, 1] > 0) & (buf[:, 0] < np.uint64(2 ** 63))
x = buf[ok].astype(np.float64)
x = x[np.argsort(x[:, 0])]
att = (x[:, 1] - x[:, 0]) / 1e3
gap = (x[1:, 0] - x[:-1, 1]) / 1e3
plan = (x[:, 3] - x[:, 2]) / 1e3
print(f"{name} per_call {per_call}: {len(x)} calls, step {step_ms:.1f} ms (events), "
      f"first start -> last exit {(x[-1, 1] - x[0, 0]) / 1e6:.1f} ms")
for nm, v in (("attention span us", att), ("gap to next call us", gap), ("k_plan span us", plan)):
    print(f"  {nm:22s} mean {v.mean():8.2f} p10 {np.percentile(v, 10):8.2f} p50 {np.median(v):8.2f} "
          f"p90 {np.percentile(v, 90):8.2f} max {v.max():8.2f} sum {v.sum() / 1e3:9.2f} ms")
big = gap > 20
print(f"  gaps > 20 us: {int(big.sum())} (sum {gap[big].sum() / 1e3:.2f} ms) -- forks / installs")
print(f"  k_plan end - previous attention exit: p50 {np.median((x[1:, 3] - x[:-1, 1]) / 1e3):.2f} us; "
      f"attention start - k_plan end p50 {np.median((x[1:, 0] - x[1:, 3]) / 1e3):.2f} us")
# the last call's CTAs (TTS_CTA: start / loop end / exit, units | smid << 32)
tb = np.zeros(2 * 1024 * 8 + 4096 * 4, dtype=np.int64)
L.tts_debug_read_trace(tb.ctypes.data_as(ctypes.c_void_p))
cta = tb[2 * 1024 * 8:].reshape(4096, 4)
cta = cta[cta[:, 0] > 0]
st0, st, ex = cta[:, 0] / 1e3, cta[:, 1] / 1e3, cta[:, 2] / 1e3  # st: after the plan wait
un = cta[:, 3] & 0xffffffff
dur = ex - st
print(f"  last call: {len(cta)} CTAs, units/CTA median {int(np.median(un))}, duration median {np.median(dur):.1f} us "
      f"(min {dur.min():.1f}, max {dur.max():.1f}), us per unit {np.median(dur / np.maximum(un, 1)):.3f}; "
      f"resident spread {st0.max() - st0.min():.1f} us, work-start spread {st.max() - st.min():.1f} us, "
      f"exit spread {ex.max() - ex.min():.1f} us")
# per-CTA dump of the last call (blockIdx order): smid, units, duration
ids = np.nonzero(tb[2 * 1024 * 8:].reshape(4096, 4)[:, 0] > 0)[0]
np.savetxt(os.path.join(ROOT, "gpurun_out", f"cta_{name}.txt"),
           np.stack([ids, cta[:, 3] >> 32, un, dur, st - st.min()], 1), fmt="%.2f",
           header="blockIdx smid units duration_us start_us")
