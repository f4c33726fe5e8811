#!/bin/bash
# ncu evidence for one configuration (run on the GPU box, from the repo root):
#   tools/profile_round.sh <config> <rotate> <tag> <attn_launch_index> <launch_skip> <launch_count>
# 1. bench line + per-call algorithmic bytes (--dump-call-bytes)
# 2. launch list of libtts kernels (one metric, --clock-control none) over a
#    window of launches past the warm-up (the timed step)
# 3. one `ncu --set full` capture of attention launch #<attn_launch_index>
# Summarise here with tools/profile_summary.py.
set -u
cfg=$1; rot=$2; tag=$3; sidx=$4; lskip=$5; lcount=$6
mkdir -p gpurun_out
args="--config $cfg --rotate $rot --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
python bench.py $args --dump-call-bytes gpurun_out/${tag}_${cfg}_callbytes.json > gpurun_out/${tag}_${cfg}_bench.json 2> gpurun_out/${tag}_${cfg}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --launch-skip $lskip -c $lcount --csv \
    --log-file gpurun_out/${tag}_${cfg}_launches.csv python bench.py $args > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_tree_umma -s $sidx -c 1 -f \
    -o gpurun_out/${tag}_${cfg}_full python bench.py --config $cfg --rotate $rot --steps 1 --warmup 1 --e2e-steps 0 \
    --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out | grep ${tag}_${cfg}
