"""Small workloads for compute-sanitizer (racecheck / synccheck / memcheck):
C1 (mma.sync path) and a C3-shaped run (tcgen05 path: d = 128, G = 7, 64
beams, whole tiles + stream-K split tiles), both through the C-ABI.
usage: compute-sanitizer --tool racecheck python tools/sanitize.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_00195_b200.runner import BeamStepRunner  # noqa: E402
from synth import workload  # noqa: E402


def main():
    for cfg, pages in ((workload.C1, 64),
                       (workload.C3.with_(L=2, n_steps=2, step_len=20, prompt=40), 2000)):
        r = BeamStepRunner(cfg, num_pages=pages, gen_device="cpu")
        n = r.run()
        torch.cuda.synchronize()
        st = r.ctx.tts_device_status()
        print(f"{cfg.name}: {n} beam-steps, status {st}", flush=True)
        assert st == 0


if __name__ == "__main__":
    main()
