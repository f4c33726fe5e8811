#!/bin/bash
# compute-sanitizer logs of tools/sanitize.py (C1 mma.sync path + C3-shaped tcgen05 path)
tag=${1:-san}
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 30 python tools/sanitize.py > gpurun_out/${tag}_sanitize_${tool}.log 2>&1
  echo "exit $?" >> gpurun_out/${tag}_sanitize_${tool}.log
done
