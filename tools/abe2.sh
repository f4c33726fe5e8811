#!/bin/bash
# env A/B over configs: tools/abe2.sh <tag> "<configs>" "<ENV=V ...>" ...
tag=$1; cfgs=$2; shift 2
mkdir -p gpurun_out
python -c "from paper_2509_00195_b200 import build; build.build(force=True)" > /dev/null 2>&1
i=0
for envs in "$@"; do
  echo "$envs" > gpurun_out/${tag}_e${i}_env.txt
  env TTS_DUMMY=1 $envs timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "random_small or c3_full or split or hybrid" > gpurun_out/${tag}_e${i}_tests.log 2>&1
  echo "pytest exit $?" >> gpurun_out/${tag}_e${i}_tests.log
  for c in $cfgs; do
    env TTS_DUMMY=1 $envs timeout 900 python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_e${i}_$c.json 2> gpurun_out/${tag}_e${i}_$c.err
  done
  i=$((i+1))
done
exit 0
