#!/bin/bash
# confirmation at HEAD: GPU suite, smoke, default bench line (C3), C2 line
tag=${1:-conf}
mkdir -p gpurun_out
python -c "from paper_2509_00195_b200 import build; build.build(force=True)" > gpurun_out/${tag}_build.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/${tag}_gpu_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/${tag}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${tag}_bench_default.json 2> gpurun_out/${tag}_bench_default.err
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/${tag}_bench_C2.json 2> gpurun_out/${tag}_bench_C2.err
exit 0
