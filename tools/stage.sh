#!/bin/bash
# staged GPU check: quick parity subset (bail out on failure/hang), then full gpu tests, bench lines, traces
tag=$1
mkdir -p gpurun_out
timeout 200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c1_full or random_small or c2_full or c3_full" > gpurun_out/${tag}_quick.log 2>&1
rc=$?; echo "quick rc=$rc" >> gpurun_out/${tag}_quick.log
[ $rc -ne 0 ] && exit 0
timeout 700 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${tag}_tests.log
for cfg in C2 C3; do
  timeout 300 python bench.py --config $cfg --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_bench_$cfg.json 2> gpurun_out/${tag}_bench_$cfg.err
done
python tools/bench_summary.py gpurun_out/${tag}_bench_C2.json gpurun_out/${tag}_bench_C3.json > gpurun_out/${tag}_summary.txt 2>&1
if [ -n "$2" ]; then
  timeout 300 python tools/trace.py 3 C2 > gpurun_out/${tag}_trace_c2.txt 2>&1
  timeout 400 python tools/trace.py 6 C3 > gpurun_out/${tag}_trace_c3.txt 2>&1
fi
exit 0
