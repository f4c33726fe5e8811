#!/bin/bash
# A/B of libtts build variants: tools/abv.sh <tag> "<flags A>" "<flags B>" ...
# per variant: build with NVCC_EXTRA, C3 and C2 bench lines (short), a parity smoke
tag=$1; shift
mkdir -p gpurun_out
i=0
for flags in "$@"; do
  NVCC_EXTRA="$flags" python -c "from paper_2509_00195_b200 import build; build.build(force=True)" > gpurun_out/${tag}_v${i}_build.log 2>&1
  echo "$flags" > gpurun_out/${tag}_v${i}_flags.txt
  timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "c1_full or c3_full" > gpurun_out/${tag}_v${i}_tests.log 2>&1
  echo "pytest exit $?" >> gpurun_out/${tag}_v${i}_tests.log
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_v${i}_C3.json 2> gpurun_out/${tag}_v${i}_C3.err
  timeout 300 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_v${i}_C2.json 2> gpurun_out/${tag}_v${i}_C2.err
  i=$((i+1))
done
python -c "from paper_2509_00195_b200 import build; build.build(force=True)" > /dev/null 2>&1
exit 0
