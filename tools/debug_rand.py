import math, random, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from synth import workload
from oracle.run import OracleRun, default_num_pages
from paper_2509_00195_b200.runner import BeamStepRunner

def cfg_for(seed):
    rnd = random.Random(seed)
    Hkv = rnd.choice([1, 2]); G = rnd.choice([1, 2, 4, 6, 7, 8, 16]); N = rnd.choice([4, 8, 16, 32, 64])
    M = rnd.choice([m for m in (2, 4, 8) if N % m == 0])
    return workload.Config(f"rand{seed}", R=rnd.choice([1, 2, 3]), N=N, M=M, L=rnd.choice([1, 2, 3]),
                          Hq=G * Hkv, Hkv=Hkv, d=rnd.choice([64, 128]), P=16,
                          prompt=rnd.choice([0, 5, 16, 37, 100]), n_steps=4, step_len=0,
                          ln_mu=math.log(rnd.choice([5, 20, 40])), ln_sigma=1.0, ln_cap=80,
                          seed=7000 + seed, q_scale=rnd.choice([1.0, 4.0]), fine_scores=rnd.random() < 0.5)

for seed in [int(x) for x in sys.argv[1:]]:
    cfg = cfg_for(seed)
    np_ = default_num_pages(cfg, cfg.R)
    orc = OracleRun(cfg, num_pages=np_)
    samp = lambda it: [(r, b, 0) for r in it.reqs for b in range(cfg.N)] if it.t < 2 else []
    tr = orc.run(sample=samp, max_iters=2)
    run = BeamStepRunner(cfg, num_pages=np_)
    outs = {}
    def on_iter(it, out, active):
        if it.t < 2:
            outs[it.t] = out.clone().cpu()
    run.run(on_iter=on_iter, max_iters=2)
    o = outs[0]
    print(cfg)
    print("nan rows t0:", torch.isnan(o[0]).any(-1).nonzero().tolist()[:20])
    ref = tr.outputs[(0, 0, 0, 0)]
    print("gpu b0 h0", o[0, 0, 0, 0, :6].tolist())
    print("ref b0 h0", ref[0, :6].tolist())
    for b in range(min(cfg.N, 4)):
        for h in range(cfg.Hq):
            r = tr.outputs[(0, 0, b, 0)][h]
            g = o[0, 0, b, h].double().numpy()
            print(b, h, float(np.abs(g - r).max() / np.abs(r).max()))
