python -c "from paper_2509_00195_b200 import build; build.build(force=True)" > /dev/null 2>&1
python tools/prof.py C3 3 > gpurun_out/q2_prof_c3.log 2>&1
TTS_POLY=1 python tools/prof.py C3 3 > gpurun_out/q2_prof_c3_p1.log 2>&1
TTS_POLY=2 python tools/prof.py C3 3 > gpurun_out/q2_prof_c3_p2.log 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/q2_bench_C3.json 2> gpurun_out/q2_bench_C3.err
TTS_POLY=2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/q2p_bench_C3.json 2> gpurun_out/q2p_bench_C3.err
TTS_POLY=1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/q2q_bench_C3.json 2> gpurun_out/q2q_bench_C3.err
