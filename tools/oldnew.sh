mkdir -p gpurun_out
for c in C3 C2 C4; do
  a="--config $c --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0"
  [ $c = C4 ] && a="--config $c --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0"
  timeout 900 python bench.py $a > gpurun_out/on_new_$c.json 2>/dev/null
  (cd old_head && timeout 900 python bench.py $a > ../gpurun_out/on_old_$c.json 2>/dev/null)
done
timeout 900 python bench.py --config C5 --tts-steps 8 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/on_new_C5.json 2>/dev/null
(cd old_head && timeout 900 python bench.py --config C5 --tts-steps 8 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > ../gpurun_out/on_old_C5.json 2>/dev/null)
