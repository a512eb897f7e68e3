#!/bin/bash
# Tensor-core MNIST kernel: phase trace + ncu capture. Usage: bash scripts/gpu_tc.sh <tag>
TAG=${1:-tc}; OUT=gpurun_out/$TAG; mkdir -p $OUT
PGB_TRACE=1 python paper_2010_09063_b200/build.py > $OUT/trace_build.log 2>&1
timeout 300 python scripts/trace_phases.py > $OUT/trace.txt 2>&1
cat $OUT/trace.txt
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:tc_kernel|fused_kernel|aggregate_kernel" -s 10 -c 4 \
   -o $OUT/prof python bench.py --model mnist_cnn --steps 10 --warmup 3 --no-cpu-baseline > $OUT/ncu_full.log 2>&1
tail -n 3 $OUT/ncu_full.log
