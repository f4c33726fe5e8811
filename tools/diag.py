"""Quick device diagnostics: attention kernel in use, HBM read / copy bandwidth,
C3-shaped decode-call time."""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_00195_b200 import build  # noqa: E402

build.build()
from paper_2509_00195_b200 import tts  # noqa: E402
from paper_2509_00195_b200.runner import BeamStepRunner  # noqa: E402
from synth import workload  # noqa: E402

dev = torch.device("cuda", 0)
buf = torch.empty(4 << 30, dtype=torch.uint8, device=dev)
buf.fill_(1)
os.environ["TTS_PROBE_VERBOSE"] = "1"
print("read GB/s", [round(tts.stream_read_gbs(buf, 10)) for _ in range(3)])
x = buf.view(torch.float32)
x.fill_(1.0)
for _ in range(2):
    x.sum()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    x.sum()
e1.record()
torch.cuda.synchronize()
print("torch sum read GB/s", round(x.numel() * 4 * 10 / (e0.elapsed_time(e1) / 1e3) / 1e9))
a = torch.empty(1 << 30, dtype=torch.bfloat16, device=dev)
b = torch.empty_like(a)
for _ in range(3):
    b.copy_(a)
e0.record()
for _ in range(10):
    b.copy_(a)
e1.record()
torch.cuda.synchronize()
print("copy GB/s", round(2 * a.numel() * 2 * 10 / (e0.elapsed_time(e1) / 1e3) / 1e9))
del buf, a, b
cfg = workload.C3.with_(n_steps=2)
r = BeamStepRunner(cfg, gen_device=None)
print("attention kernel:", r.ctx.attention_kernel(), "occupancy probe in ctx")
t0 = time.time()
r.run()
torch.cuda.synchronize()
r.release()
e0.record()
n = r.run()
e1.record()
torch.cuda.synchronize()
print(f"C3 2-step run: {e0.elapsed_time(e1):.1f} ms for {n} beam-steps -> {n / (e0.elapsed_time(e1) / 1e3):.0f} beam-steps/s (incl. input gen)")
