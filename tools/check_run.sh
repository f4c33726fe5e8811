#!/bin/bash
# device-side bounds checks (TTS_CHECK build: traps on a violated schedule
# index) over the GPU parity / edge / spec / dist tests, default and pair mode
tag=${1:-chk}
mkdir -p gpurun_out
NVCC_EXTRA="-DTTS_CHECK" python -c "from paper_2509_00195_b200 import build; build.build(force=True)" > gpurun_out/${tag}_build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/${tag}_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/${tag}_tests.log
TTS_PAIR=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "c3_full or c4 or c5 or random_small or split" > gpurun_out/${tag}_pair_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/${tag}_pair_tests.log
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_bench_C3.json 2> gpurun_out/${tag}_bench_C3.err
echo "bench exit $?" >> gpurun_out/${tag}_bench_C3.err
python -c "from paper_2509_00195_b200 import build; build.build(force=True)" > /dev/null 2>&1
exit 0
