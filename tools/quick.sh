#!/bin/bash
# quick GPU check: parity tests, C2/C3 bench lines (no CPU baseline), optional trace
mkdir -p gpurun_out
tag=${1:-q}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${tag}_tests.log
for cfg in C2 C3; do
  timeout 300 python bench.py --config $cfg --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_bench_$cfg.json 2> gpurun_out/${tag}_bench_$cfg.err
done
[ -n "$2" ] && timeout 400 python tools/trace.py 6 C3 > gpurun_out/${tag}_trace_c3.txt 2>&1
python tools/bench_summary.py gpurun_out/${tag}_bench_C2.json gpurun_out/${tag}_bench_C3.json > gpurun_out/${tag}_summary.txt 2>&1
exit 0
