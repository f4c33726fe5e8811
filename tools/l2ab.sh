bash tools/abe3.sh ab16 "--steps 2 --warmup 3" "TTS_L2HINT=0" "TTS_L2HINT=1 TTS_L2PERSIST_MB=32" "TTS_L2HINT=1 TTS_L2PERSIST_MB=64" "TTS_L2HINT=1 TTS_L2PERSIST_MB=96"
for mb in 0 64; do
  TTS_L2PERSIST_MB=$mb ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_tree_umma -s 3000 -c 2 --csv python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab16_ncu_$mb.csv 2>/dev/null
done
python -c "import torch; p=torch.cuda.get_device_properties(0); print('persisting L2 max', getattr(p,'persisting_l2_cache_max_size',None), 'L2', p.L2_cache_size)" > gpurun_out/ab16_props.txt 2>&1
