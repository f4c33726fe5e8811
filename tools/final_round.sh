#!/bin/bash
# end-of-round evidence on the GPU box: default bench line (C2, CPU baseline, e2e),
# reference arm, C3/C4/C5 lines, ncu launch lists + full captures for C2 and C3, smoke
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/f_bench_default.json 2> gpurun_out/f_bench_default.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f_bench_ref.json 2> gpurun_out/f_bench_ref.err
timeout 300 python bench.py --config C3 --no-cpu-baseline > gpurun_out/f_bench_C3.json 2> gpurun_out/f_bench_C3.err
timeout 400 python bench.py --config C4 --no-cpu-baseline --e2e-steps 0 --steps 1 > gpurun_out/f_bench_C4.json 2> gpurun_out/f_bench_C4.err
timeout 600 python bench.py --config C5 --no-cpu-baseline --e2e-steps 0 --steps 1 --warmup 3 --tts-steps 8 > gpurun_out/f_bench_C5.json 2> gpurun_out/f_bench_C5.err
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1
timeout 900 bash tools/profile_round.sh C2 8 r1b 20000 80000 3000
timeout 900 bash tools/profile_round.sh C3 2 r1b 10000 40000 3000
exit 0
