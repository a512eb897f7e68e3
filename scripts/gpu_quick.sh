#!/bin/bash
# Quick GPU iteration: parity tests + a short bench. Usage: bash scripts/gpu_quick.sh <tag> [model] [pytest -k expr]
TAG=${1:-q}; MODEL=${2:-mnist_cnn}; K=${3:-}
OUT=gpurun_out/$TAG; mkdir -p $OUT
if [ -n "$K" ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > $OUT/pytest_gpu.log 2>&1
else timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; fi
echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -n 15 $OUT/pytest_gpu.log
timeout 600 python bench.py --model $MODEL --steps 500 --warmup 10 --no-cpu-baseline > $OUT/bench_$MODEL.json 2> $OUT/bench_$MODEL.err
tail -n 5 $OUT/bench_$MODEL.err
python -c "import json;d=json.load(open('$OUT/bench_$MODEL.json'));print('value',d['value'],'e2e',d['e2e']['value'],'kernels_us',d['kernels_us'])"
