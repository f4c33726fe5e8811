#!/bin/bash
# quick GPU iteration: parity subset, C3 trace, C3/C2 bench, and the same bench
# with libtts built with extra flags ($2, e.g. -DTTS_WAIT_NOHINT) as variant "b"
tag=${1:-q}
extra=${2:-}
mkdir -p gpurun_out
python -c "from paper_2509_00195_b200 import build; build.build(force=True)" > gpurun_out/${tag}_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "c1_full or random_small or split or hybrid or selection or c3_full" > gpurun_out/${tag}_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/${tag}_tests.log
timeout 300 python tools/trace.py 8 C3 > gpurun_out/${tag}_trace_c3.log 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_bench_C3.json 2> gpurun_out/${tag}_bench_C3.err
timeout 300 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_bench_C2.json 2> gpurun_out/${tag}_bench_C2.err
if [ -n "$extra" ]; then
  NVCC_EXTRA="$extra" python -c "from paper_2509_00195_b200 import build; build.build(force=True)" > gpurun_out/${tag}b_build.log 2>&1
  timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "c1_full or c3_full" > gpurun_out/${tag}b_tests.log 2>&1
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}b_bench_C3.json 2> gpurun_out/${tag}b_bench_C3.err
  timeout 300 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}b_bench_C2.json 2> gpurun_out/${tag}b_bench_C2.err
fi
exit 0
