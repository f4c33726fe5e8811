#!/bin/bash
# A/B of an env toggle: tools/ab.sh <tag> <VAR> <v1> <v2> ; C2 + C3 bench lines for each value
tag=$1; var=$2; shift 2
mkdir -p gpurun_out
for val in "$@"; do
  for cfg in C2 C3; do
    env $var=$val timeout 300 python bench.py --config $cfg --no-cpu-baseline --e2e-steps 0 --steps 2 > gpurun_out/${tag}_${val}_$cfg.json 2> gpurun_out/${tag}_${val}_$cfg.err
  done
done
for val in "$@"; do python tools/bench_summary.py gpurun_out/${tag}_${val}_C2.json gpurun_out/${tag}_${val}_C3.json; done > gpurun_out/${tag}_ab.txt 2>&1
