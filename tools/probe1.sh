mkdir -p gpurun_out
python -c "from paper_2509_00195_b200 import build; build.build(force=True)" > gpurun_out/p1_build.log 2>&1
timeout 300 python tools/trace.py 3 C3 > gpurun_out/p1_trace_c3.log 2>&1
timeout 300 python tools/prof.py C3 3 > gpurun_out/p1_prof_c3.log 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/p1_bench_C3.json 2> gpurun_out/p1_bench_C3.err
exit 0
