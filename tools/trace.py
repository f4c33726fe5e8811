"""Build libtts with -DTTS_TRACE, run C3 positions, print per-unit timeline of one CTA."""
import ctypes, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2509_00195_b200 import build
lib = build.LIB.replace("libtts.so", "libtts_trace.so")
cmd = [build.NVCC, *build.ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC", "-DTTS_TRACE", *(["-DTTS_NOEXP"] if os.environ.get("NOEXP") else []),
       "-I", os.path.join(build.ROOT, "include"), "-o", lib, *build.sources()]
subprocess.run(cmd, check=True)
from paper_2509_00195_b200 import tts
tts.LIB_PATH = lib
from paper_2509_00195_b200.runner import BeamStepRunner
from synth import workload
name = sys.argv[2] if len(sys.argv) > 2 else "C3"
cfg = workload.CONFIGS[name].with_(n_steps=int(sys.argv[1]) if len(sys.argv) > 1 else 6)
r = BeamStepRunner(cfg)
r.run()
import torch; torch.cuda.synchronize()
buf = np.zeros(2 * 1024 * 8 + 4096 * 4, dtype=np.int64)
L = tts.load()
L.tts_debug_read_trace(buf.ctypes.data_as(ctypes.c_void_p))
trr = buf[:2 * 1024 * 8].reshape(2, 1024, 8)
tr, t2 = trr[0], trr[1]
cta = buf[2 * 1024 * 8:].reshape(4096, 4)
cta = cta[cta[:, 0] > 0]
if len(cta):
    t0c = cta[:, 0].min()
    st, le, ex = (cta[:, 0] - t0c) / 1e3, (cta[:, 1] - t0c) / 1e3, (cta[:, 2] - t0c) / 1e3
    un = cta[:, 3] & 0xffffffff
    sm = cta[:, 3] >> 32
    print(f"last launch: {len(cta)} CTAs, span {ex.max():.1f} us; start min/med/max {st.min():.1f}/{np.median(st):.1f}/{st.max():.1f};"
          f" exit min/med/max {ex.min():.1f}/{np.median(ex):.1f}/{ex.max():.1f}; units min/med/max {un.min()}/{int(np.median(un))}/{un.max()}")
    dur = ex - st
    print(f"  CTA duration min/med/max {dur.min():.1f}/{np.median(dur):.1f}/{dur.max():.1f} us; us per unit (median) {np.median(dur / np.maximum(un, 1)):.3f};"
          f" epilogue (exit - loop end) median {np.median(ex - le):.2f} us; distinct SMs {len(set(sm.tolist()))}")
    hist = np.histogram(ex, bins=10)
    print("  exit-time histogram:", hist[0].tolist(), "edges", [round(x, 1) for x in hist[1].tolist()])
n = int((tr[:, 4] > 0).sum())
t0 = tr[0, 4]
print("units", n)
e = tr[1023]
print("CTA: start->prologue", e[1] - e[0], "prologue->loop end", e[2] - e[1], "loop end->exit", e[3] - e[2], "total", e[3] - e[0])
print("j: mma_fullwait_start mma_fullwait_end mma_pfull_end mma_pv_commit | sm_wait_start sm_sfull_end sm_arrive (cycles rel)")
for j in range(min(n, 40)):
    e = tr[j] - t0
    print(j, e[0], e[1], e[2], e[3], "|", e[4], e[5], e[6], " softmax_busy", tr[j, 6] - tr[j, 5], " waitS", tr[j, 5] - tr[j, 4])
tr[1023] = 0
d = tr[1:n, 5] - tr[:n - 1, 5]
print("median cycles per unit", np.median(d), "softmax busy median", np.median(tr[:n, 6] - tr[:n, 5]),
      "sfull wait median", np.median(tr[:n, 5] - tr[:n, 4]), "mma pfull-wait median", np.median(tr[:n, 2] - tr[:n, 1]))

print("per-warp P arrive (rel. to warp 0) and MMA pfull_end (rel. to last warp), first 12 units:")
for j in range(min(n, 12)):
    a = t2[j, :4]
    print(j, [int(x - a[0]) for x in a], "mma_pfull_end - last_arrive", int(tr[j, 2] - a.max()))
print("median S-issue cycles (fullwait_end -> issue_s done):", np.median(tr[:n-1, 7] - tr[:n-1, 1]),
      " issue_s done -> pfull_end:", np.median(tr[:n-1, 2] - tr[:n-1, 7]), " pfull_end -> pv_commit:", np.median(tr[:n-1, 3] - tr[:n-1, 2]),
      " pv_commit -> next fullwait_start:", np.median(tr[1:n, 0] - tr[:n-1, 3]))
d = t2[:n, :4] - t2[:n, :1]
print("median arrive offsets vs warp 0:", np.median(d, axis=0), " median pfull_end - last arrive:", np.median(tr[:n, 2] - t2[:n, :4].max(1)))
full = []
print("member units", len(full), "of", n)
if full:
    f = np.array(full)
    print("member path medians: meta->ld", np.median(t2[f, 1] - t2[f, 0]), "ld->max", np.median(t2[f, 2] - t2[f, 1]),
          "max->exp_done", np.median(t2[f, 3] - t2[f, 2]), "exp->st_done", np.median(t2[f, 4] - t2[f, 3]),
          "st->arrive", np.median(tr[f, 6] - t2[f, 4]), "sfull->meta", np.median(t2[f, 0] - tr[f, 5]),
          "rescales", int((t2[f, 7] > 0).sum()))
sk = [j for j in range(n) if t2[j, 3] == 0]
if sk:
    s_ = np.array(sk)
    print("skip path medians: sfull->meta", np.median(t2[s_, 0] - tr[s_, 5]), "meta->st_done", np.median(t2[s_, 4] - t2[s_, 0]),
          "st->arrive", np.median(tr[s_, 6] - t2[s_, 4]))
