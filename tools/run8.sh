mkdir -p gpurun_out
for cfg in C2 C3; do timeout 300 python bench.py --config $cfg --no-cpu-baseline --e2e-steps 0 > gpurun_out/p4_bench_$cfg.json 2> gpurun_out/p4_bench_$cfg.err; done
python tools/bench_summary.py gpurun_out/p4_bench_C2.json gpurun_out/p4_bench_C3.json > gpurun_out/p4_summary.txt 2>&1
timeout 300 python tools/trace.py 3 C2 > gpurun_out/p4_trace_c2.txt 2>&1
timeout 400 python tools/trace.py 6 C3 > gpurun_out/p4_trace_c3.txt 2>&1
