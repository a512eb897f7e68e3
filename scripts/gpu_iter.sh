#!/bin/bash
# Iteration loop for the MNIST kernel: MNIST parity tests, short bench, phase trace.
# Usage: bash scripts/gpu_iter.sh <tag> [pytest -k expr]
TAG=${1:-it}; K=${2:-mnist or tc_gpu or umma}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q -k "$K" > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -n 4 $OUT/pytest_gpu.log
timeout 300 python bench.py --model mnist_cnn --steps 500 --warmup 10 --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
python -c "import json;d=json.load(open('$OUT/bench.json'));print('value',round(d['value']),'e2e',round(d['e2e']['value']),'kernels_us',d['kernels_us'])"
PGB_TRACE=1 python paper_2010_09063_b200/build.py > /dev/null 2>&1
timeout 300 python scripts/trace_phases.py > $OUT/trace.txt 2>&1; cat $OUT/trace.txt
