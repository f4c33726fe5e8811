#!/bin/bash
# end-of-round evidence on the GPU box (run under gpurun from the repo root):
# full GPU suite, smoke, the default bench line (C3: cpu_baseline + e2e), the
# reference arm, C2 / C4 / C5 lines, speculation on/off, ncu launch lists and
# full captures of C3 and C2 (compute-sanitizer is closed on this pool)
tag=${1:-r2f}
mkdir -p gpurun_out
python -c "from paper_2509_00195_b200 import build; build.build(force=True)" > gpurun_out/${tag}_build.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/${tag}_gpu_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/${tag}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${tag}_bench_default.json 2> gpurun_out/${tag}_bench_default.err
timeout 400 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/${tag}_bench_C2.json 2> gpurun_out/${tag}_bench_C2.err
timeout 600 python bench.py --config C4 --no-cpu-baseline --e2e-steps 0 --steps 1 > gpurun_out/${tag}_bench_C4.json 2> gpurun_out/${tag}_bench_C4.err
timeout 900 python bench.py --config C5 --no-cpu-baseline --e2e-steps 0 --steps 1 --tts-steps 8 > gpurun_out/${tag}_bench_C5.json 2> gpurun_out/${tag}_bench_C5.err
timeout 900 python bench.py --config C5 --no-cpu-baseline --e2e-steps 0 --steps 1 > gpurun_out/${tag}_bench_C5full.json 2> gpurun_out/${tag}_bench_C5full.err
timeout 900 python tools/spec_bench.py 2 64 4 28 > gpurun_out/${tag}_spec_bench.json 2> gpurun_out/${tag}_spec_bench.err
timeout 1500 bash tools/profile_round.sh C3 1 ${tag} 3000 6000 400 > gpurun_out/${tag}_prof_C3.log 2>&1
timeout 1500 bash tools/profile_round.sh C2 32 ${tag} 1500 3000 400 > gpurun_out/${tag}_prof_C2.log 2>&1
exit 0
