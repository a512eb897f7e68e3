#!/bin/bash
# ncu evidence for one model: launch list + full capture of the named kernels.
# Usage: bash scripts/gpu_prof.sh <tag> <model> <kernel-regex>
TAG=${1:-r01}; MODEL=${2:-mnist_cnn}; KRE=${3:-tc_kernel|fused_kernel|aggregate_kernel}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 200 --csv \
   --log-file $OUT/launches_$MODEL.csv python bench.py --model $MODEL --steps 30 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_$MODEL.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$KRE" -s 10 -c 4 \
   -o $OUT/prof_$MODEL python bench.py --model $MODEL --steps 10 --warmup 3 --no-cpu-baseline > $OUT/ncu_full_$MODEL.log 2>&1
tail -n 3 $OUT/ncu_full_$MODEL.log
