#!/bin/bash
# CIFAR step launch list under ncu with extra env. Usage: bash scripts/cifar_launches_env.sh <tag> [ENV=VAL ...]
TAG=${1:-cl}; shift; mkdir -p gpurun_out
env "$@" timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 150 -c 200 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --model cifar_cnn --steps 6 --warmup 3 \
  --epochs 1 --no-cpu-baseline > /dev/null 2>&1
python scripts/step_launches.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_step.txt
