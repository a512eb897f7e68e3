#!/bin/bash
# One bench line per BASELINE config (device + e2e), short runs.
OUT=gpurun_out/${1:-all}; mkdir -p $OUT
for M in mnist_cnn cifar_cnn fcnn logreg embed; do
  timeout 600 python bench.py --model $M --steps ${2:-200} --warmup 5 --no-cpu-baseline > $OUT/$M.json 2> $OUT/$M.err
  python -c "import json;d=json.load(open('$OUT/$M.json'));print('$M', round(d['value']), 'e2e', round(d['e2e']['value']), 'ms/step', round(d['ms_per_step'],4), d['kernels_us'])" || tail -3 $OUT/$M.err
done
