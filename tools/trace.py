"""Build libtts with -DTTS_TRACE, run C3 positions, print per-unit timeline of one CTA."""
import ctypes, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2509_00195_b200 import build
lib = build.LIB.replace("libtts.so", "libtts_trace.so")
cmd = [build.NVCC, *build.ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC", "-DTTS_TRACE",
       "-I", os.path.join(build.ROOT, "include"), "-o", lib, *build.sources()]
subprocess.run(cmd, check=True)
from paper_2509_00195_b200 import tts
tts.LIB_PATH = lib
from paper_2509_00195_b200.runner import BeamStepRunner
from synth import workload
cfg = workload.C3.with_(n_steps=int(sys.argv[1]) if len(sys.argv) > 1 else 6)
r = BeamStepRunner(cfg)
r.run()
import torch; torch.cuda.synchronize()
tr = np.zeros((1024, 8), dtype=np.int64)
L = tts.load()
L.tts_debug_read_trace(tr.ctypes.data_as(ctypes.c_void_p))
n = int((tr[:, 4] > 0).sum())
t0 = tr[0, 4]
print("units", n)
print("j: mma_fullwait_start mma_fullwait_end mma_pfull_end mma_pv_commit | sm_wait_start sm_sfull_end sm_arrive (cycles rel)")
for j in range(min(n, 40)):
    e = tr[j] - t0
    print(j, e[0], e[1], e[2], e[3], "|", e[4], e[5], e[6], " softmax_busy", tr[j, 6] - tr[j, 5], " waitS", tr[j, 5] - tr[j, 4])
d = tr[1:n, 5] - tr[:n - 1, 5]
print("median cycles per unit", np.median(d), "softmax busy median", np.median(tr[:n, 6] - tr[:n, 5]),
      "sfull wait median", np.median(tr[:n, 5] - tr[:n, 4]), "mma pfull-wait median", np.median(tr[:n, 2] - tr[:n, 1]))
