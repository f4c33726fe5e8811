for sc in 2 3 1; do
  TTS_SCHED=$sc ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:k_tree_umma -s 3000 -c 2 --csv python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/sched_ncu_$sc.csv 2>/dev/null
done
