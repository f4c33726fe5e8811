#!/bin/bash
# quick GPU iteration: profile split (TTS_PROF), C3 + C2 bench lines, a parity subset
tag=${1:-q}
mkdir -p gpurun_out
python -c "from paper_2509_00195_b200 import build; build.build(force=True)" > gpurun_out/${tag}_build.log 2>&1
python tools/prof.py C3 3 > gpurun_out/${tag}_prof_c3.log 2>&1
python tools/prof.py C2 3 > gpurun_out/${tag}_prof_c2.log 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_bench_C3.json 2> gpurun_out/${tag}_bench_C3.err
python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_bench_C2.json 2> gpurun_out/${tag}_bench_C2.err
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "c3_full or random_small or split or hybrid or c1_full" > gpurun_out/${tag}_tests.log 2>&1
exit 0
