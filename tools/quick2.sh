#!/bin/bash
# quick GPU iteration (variant A/B): parity subset, C3 prof + bench, C3 bench with TTS_POLY=1, C2 bench
tag=${1:-q}
mkdir -p gpurun_out
python -c "from paper_2509_00195_b200 import build; build.build(force=True)" > gpurun_out/${tag}_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "c1_full or random_small or split or hybrid or selection or c3_full" > gpurun_out/${tag}_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/${tag}_tests.log
timeout 300 python tools/prof.py C3 3 > gpurun_out/${tag}_prof_c3.log 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_bench_C3.json 2> gpurun_out/${tag}_bench_C3.err
TTS_POLY=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_bench_C3p1.json 2> gpurun_out/${tag}_bench_C3p1.err
timeout 300 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_bench_C2.json 2> gpurun_out/${tag}_bench_C2.err
exit 0
