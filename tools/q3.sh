python -c "from paper_2509_00195_b200 import build; build.build(force=True)" > /dev/null 2>&1
TTS_CTAS_PER_SM=1 python tools/prof.py C3 3 > gpurun_out/q3_prof_c3_1cta.log 2>&1
TTS_CTAS_PER_SM=1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/q3_bench_C3.json 2> gpurun_out/q3_bench_C3.err
