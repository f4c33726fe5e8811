#!/bin/bash
# one GPU call: tests, smoke, default bench line (+ C2), sanitizer logs
# usage (under gpurun): bash tools/gpu_check.sh <tag>
tag=${1:-chk}
mkdir -p gpurun_out
python -c "from paper_2509_00195_b200 import build; build.build(force=True)" > gpurun_out/${tag}_build.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x --durations=15 > gpurun_out/${tag}_gpu_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/${tag}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/${tag}_bench_C3.json 2> gpurun_out/${tag}_bench_C3.err
timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_C2.json 2> gpurun_out/${tag}_bench_C2.err
for tool in racecheck synccheck memcheck; do
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py > gpurun_out/${tag}_sanitize_${tool}.log 2>&1
  echo "exit $?" >> gpurun_out/${tag}_sanitize_${tool}.log
done
exit 0
