#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list and one full capture.
# Usage (from the repo root, under gpurun): bash scripts/gpu_check.sh [tag] [model]
TAG=${1:-r01}; MODEL=${2:-mnist_cnn}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py --model $MODEL > $OUT/bench.json 2> $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 200 --csv \
   --log-file $OUT/launches.csv python bench.py --model $MODEL --steps 30 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${NCU_K:-tc_kernel|fused_kernel|aggregate_kernel}" -s 20 -c 3 \
   -o $OUT/prof python bench.py --model $MODEL --steps 10 --warmup 3 --no-cpu-baseline > $OUT/ncu_full.log 2>&1
for f in $OUT/*.log; do tail -n 3 $f; done
cat $OUT/bench.json
