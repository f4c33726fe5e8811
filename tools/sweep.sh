#!/bin/bash
# usage: tools/sweep.sh <config> <rotate> ; prints value / achieved GB/s / us per attention launch per split setting
CFG=${1:-C2}; ROT=${2:-8}; shift 2
for s in "$@"; do
  TTS_SPLITS=$s timeout 300 python bench.py --config $CFG --steps 1 --warmup 1 --rotate $ROT --e2e-steps 0 --no-cpu-baseline > /tmp/sw.json 2>/tmp/sw.err || { echo "splits $s failed"; tail -3 /tmp/sw.err; continue; }
  python - "$s" <<'PY'
import json,sys
d=json.load(open('/tmp/sw.json')); r=d['roofline']
print(f"splits={sys.argv[1]} value={d['value']:.0f} achieved={r['achieved']:.0f}GB/s frac={r['frac']:.3f} us/launch={r['attn_ms_per_step']/r['attn_launches_per_step']*1e3:.1f} share={r['attn_share_of_step']:.2f}")
PY
done
