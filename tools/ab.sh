#!/bin/bash
# A/B of an environment toggle: parity subset + C3/C2 bench with and without it
# usage: bash tools/ab.sh <tag> "<ENV=VAL ...>"
tag=$1; envs=$2
mkdir -p gpurun_out
python -c "from paper_2509_00195_b200 import build; build.build(force=True)" > /dev/null 2>&1
env $envs timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "random_small or c3_full or split or selection" > gpurun_out/${tag}_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/${tag}_tests.log
for side in A B; do
  if [ $side = B ]; then e="$envs"; else e="TTS_DUMMY=1"; fi
  env $e timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}${side}_bench_C3.json 2>/dev/null
  env $e timeout 300 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}${side}_bench_C2.json 2>/dev/null
done
