#!/bin/bash
# A/B of environment toggles: tools/abe.sh <tag> "<ENV=V ...>" "<ENV=V ...>" ...
# per variant: parity subset, C3 and C2 bench lines (short)
tag=$1; shift
mkdir -p gpurun_out
python -c "from paper_2509_00195_b200 import build; build.build(force=True)" > /dev/null 2>&1
i=0
for envs in "$@"; do
  echo "$envs" > gpurun_out/${tag}_e${i}_env.txt
  env TTS_DUMMY=1 $envs timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "random_small or c3_full or split or hybrid" > gpurun_out/${tag}_e${i}_tests.log 2>&1
  echo "pytest exit $?" >> gpurun_out/${tag}_e${i}_tests.log
  env TTS_DUMMY=1 $envs timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_e${i}_C3.json 2> gpurun_out/${tag}_e${i}_C3.err
  env TTS_DUMMY=1 $envs timeout 300 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_e${i}_C2.json 2> gpurun_out/${tag}_e${i}_C2.err
  i=$((i+1))
done
exit 0
