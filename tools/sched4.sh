mkdir -p gpurun_out
TTS_SCHED=4 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/s4_tests.log 2>&1; echo "exit $?" >> gpurun_out/s4_tests.log
bash tools/abe3.sh s4c3 "--steps 2 --warmup 3" "TTS_SCHED=2" "TTS_SCHED=4"
bash tools/abe3.sh s4c5 "--config C5 --tts-steps 8 --steps 1 --warmup 3" "TTS_SCHED=2" "TTS_SCHED=4"
bash tools/abe3.sh s4c4 "--config C4 --steps 1 --warmup 3" "TTS_SCHED=2" "TTS_SCHED=4"
bash tools/abe3.sh s4c2 "--config C2 --steps 2 --warmup 3" "TTS_SCHED=2" "TTS_SCHED=4"
TTS_SCHED=4 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:k_tree_umma -s 3000 -c 2 --csv python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/sched_ncu_4.csv 2>/dev/null
