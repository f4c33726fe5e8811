mkdir -p gpurun_out
for pc in 4 8 16 32; do
  a="--config C2 --per-call $pc --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0"
  timeout 900 python bench.py $a > gpurun_out/pc_new_$pc.json 2>/dev/null
  (cd old_head && timeout 900 python bench.py $a > ../gpurun_out/pc_old_$pc.json 2>/dev/null)
done
