"""Build libtts with -DTTS_PROF (per-warp cycle accounting of k_tree_umma,
accumulated in registers, one write per warp at exit) and print, for the last
launch of a run, the per-unit cycle split of every warp role (median over CTAs).
usage: python tools/prof.py <config> [tts_steps] [extra nvcc -D flags...]"""
import ctypes
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2509_00195_b200 import build  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
extra = sys.argv[3:]
lib = build.LIB.replace("libtts.so", "libtts_prof.so")
cmd = [build.NVCC, *build.ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC", "-DTTS_PROF",
       *extra, "-I", os.path.join(build.ROOT, "include"), "-o", lib, *build.sources()]
subprocess.run(cmd, check=True, capture_output=True)
from paper_2509_00195_b200 import tts  # noqa: E402

tts.LIB_PATH = lib
import torch  # noqa: E402

from paper_2509_00195_b200.runner import BeamStepRunner  # noqa: E402
from synth import workload  # noqa: E402

cfg = workload.CONFIGS[name].with_(n_steps=steps)
r = BeamStepRunner(cfg)
r.run()
torch.cuda.synchronize()
buf = np.zeros(512 * 12 * 16, dtype=np.int64)
tts.load().tts_debug_read_prof(buf.ctypes.data_as(ctypes.c_void_p))
pr = buf.reshape(512, 12, 16)
n_cta = int((pr[:, 10, :].sum(1) > 0).sum())
pr = pr[:n_cta]
units = pr[:, 0, 7].astype(float)
print(f"{name} {extra}: {n_cta} CTAs, units per CTA median {np.median(units):.0f} (min {units.min():.0f}, max {units.max():.0f})")
tot = pr[:, 0, :6].sum(1) + pr[:, 0, 8:12].sum(1)
print(f"  softmax warp total cycles median {np.median(tot):.0f}  -> cycles per unit {np.median(tot / np.maximum(units, 1)):.0f}")
names = {
    "softmax": ["wait S", "member softmax", "skipped", "other", "rescale", "P store+arrive", "", "", "load Q",
                "wait last PV", "O store / partial", "merge"],
    "K producer": ["wait slot", "issue", "item loads"],
    "V producer": ["wait slot", "issue", "item loads"],
    "S": ["wait K", "wait S buf", "issue", "wait Q"],
    "PV": ["wait V", "wait P", "wait O", "issue"],
}
for w in range(8):
    x = pr[:, w, :6] / np.maximum(units, 1)[:, None]
    mem = np.median(pr[:, w, 6] / np.maximum(units, 1))
    x = pr[:, w, :12] / np.maximum(units, 1)[:, None]
    print(f"  softmax warp {w}: member fraction {mem:.2f}; " +
          ", ".join(f"{n} {np.median(x[:, k]):.0f}" for k, n in enumerate(names["softmax"]) if n))
print(f"  merges per CTA (warp 0) mean {pr[:, 0, 12].mean():.2f}")
for w, role in ((8, "K producer"), (9, "V producer"), (10, "S"), (11, "PV")):
    x = pr[:, w, :len(names[role])] / np.maximum(units, 1)[:, None]
    print(f"  {role:8s} warp {w}: " + ", ".join(f"{n} {np.median(x[:, k]):.0f}" for k, n in enumerate(names[role])))
