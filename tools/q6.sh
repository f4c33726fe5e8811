python -c "from paper_2509_00195_b200 import build; build.build(force=True)" > /dev/null 2>&1
for a in 2 3 4 6; do
  TTS_S_AHEAD=$a timeout 300 python tools/prof.py C3 3 > gpurun_out/q6_prof_c3_$a.log 2>&1
  TTS_S_AHEAD=$a timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/q6s${a}_bench_C3.json 2> /dev/null
done
