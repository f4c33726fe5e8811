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
    bid = np.nonzero(buf[2 * 1024 * 8:].reshape(4096, 4)[:, 0] > 0)[0]
    rate = dur / np.maximum(un, 1)
    print("  us per unit by CTA half: blockIdx < 148: %.3f, >= 148: %.3f" % (np.median(rate[bid < 148]), np.median(rate[bid >= 148])))
    order = np.argsort(sm)
    print("  us per unit by SM id (pairs of co-resident CTAs averaged), 16 per row:")
    per_sm = {}
    for s_, r_ in zip(sm.tolist(), rate.tolist()):
        per_sm.setdefault(s_, []).append(r_)
    ks = sorted(per_sm)
    for i in range(0, len(ks), 16):
        print("   ", " ".join(f"{np.mean(per_sm[k]):.3f}" for k in ks[i:i + 16]))
    hist = np.histogram(ex, bins=10)
    print("  exit-time histogram:", hist[0].tolist(), "edges", [round(x, 1) for x in hist[1].tolist()])
n = int((tr[:, 3] > 0).sum())
print("units traced", n)
t0 = tr[0, 0]
ev = ["S kfull", "S sbuf", "S issued", "sm0 sfull", "sm0 pair", "sm0 arrive", "PV vfull", "PV pfull"]
ev2 = ["sm5 sfull", "sm5 pair", "sm5 arrive", "Kprod slot", "Vprod slot"]
print("j | " + " ".join(f"{e:>10s}" for e in ev + ev2))
for j in list(range(0, min(n, 12))) + list(range(max(12, n // 2), min(n, n // 2 + 12))):
    print(j, "|", " ".join(f"{int(x - t0):10d}" for x in list(tr[j]) + list(t2[j, :5])))
lo, hi = max(1, n // 4), max(2, 3 * n // 4)
d = lambda a, b: np.median(a[lo:hi] - b[lo:hi])
print("median per unit period (sm0 sfull):", np.median(np.diff(tr[lo:hi, 3])))
print("median: S kfull->sbuf %.0f, sbuf->issued %.0f, issued->sm0 sfull %.0f, sm0 sfull->pair %.0f, pair->arrive %.0f,"
      " sm0 arrive->PV pfull %.0f, PV vfull(j)-> S sbuf(j+2) %.0f" % (
      d(tr[:, 1], tr[:, 0]), d(tr[:, 2], tr[:, 1]), d(tr[:, 3], tr[:, 2]), d(tr[:, 4], tr[:, 3]), d(tr[:, 5], tr[:, 4]),
      d(tr[:, 7], tr[:, 5]), np.median(tr[lo + 2:hi + 2, 1] - tr[lo:hi, 7])))
print("median sm5: sfull->pair %.0f, pair->arrive %.0f" % (d(t2[:, 1], t2[:, 0]), d(t2[:, 2], t2[:, 1])))
