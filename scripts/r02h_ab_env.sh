#!/bin/bash
# CIFAR bench A/B over env settings, interleaved. Usage: bash scripts/r02h_ab_env.sh "" "X=1" ...
for r in 1 2; do for e in "$@"; do
  env $e timeout 300 python bench.py --model cifar_cnn --steps 300 --warmup 5 --epochs 1 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.load(sys.stdin);print('[$e]', round(d['value']), 'e2e', round(d['e2e']['value']))"
done; done
