"""Cross-group duplication of a decode call's pages (product path only): run a
config through BeamStepRunner up to iteration T, read the device block tables,
and compare the distinct pages of the whole request with the sum over the
attention kernel's beam groups (16 beams for G = 7) of their distinct pages --
the factor by which a group-by-group kernel loads shared pages more than once.
usage: python tools/group_dup.py <config> <iteration> [group_beams]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2509_00195_b200.runner import BeamStepRunner  # noqa: E402
from synth import workload  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
gb = int(sys.argv[3]) if len(sys.argv) > 3 else 16
cfg = workload.CONFIGS[name]
r = BeamStepRunner(cfg)
r.run(max_iters=T)
snap = r.ctx.tts_block_table_snapshot(0, with_pool_state=False)
r.ctx.sync()
tables, lens = snap["tables"], snap["lens"]
P = cfg.P
pages = [set(int(x) for x in tables[b][: -(-int(lens[b]) // P)]) for b in range(cfg.N)]
union = set().union(*pages)
per_group = [set().union(*pages[g:g + gb]) for g in range(0, cfg.N, gb)]
s = sum(len(x) for x in per_group)
print(f"{name} iteration {T}: {len(union)} distinct pages in the request, {s} summed over "
      f"{len(per_group)} groups of {gb} beams -> duplication {s / len(union):.3f}; "
      f"mean beam length {np.mean(lens):.0f} tokens")
