#!/bin/bash
# env A/B with bench args: tools/abe3.sh <tag> "<bench args>" "<ENV=V>" ...
tag=$1; args=$2; shift 2
mkdir -p gpurun_out
python -c "from paper_2509_00195_b200 import build; build.build(force=True)" > /dev/null 2>&1
i=0
for envs in "$@"; do
  echo "$envs | $args" > gpurun_out/${tag}_e${i}_env.txt
  env TTS_DUMMY=1 $envs timeout 900 python bench.py $args --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_e${i}.json 2> gpurun_out/${tag}_e${i}.err
  i=$((i+1))
done
exit 0
