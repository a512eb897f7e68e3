#!/bin/bash
# A/B of the MNIST bench on one box: builds of other revisions (ab/lib*.so)
# against the in-tree library, interleaved.
# Usage: bash scripts/ab_bench.sh [rounds] [libs...]   (default: ab/libA.so)
R=${1:-3}; shift
LIBS=${@:-ab/libA.so}
one() {
  timeout 300 python bench.py --model mnist_cnn --steps 3000 --warmup 10 --no-cpu-baseline 2>/dev/null |
    python -c "import json,sys;d=json.load(sys.stdin);print('$1', 'value', round(d['value']), 'e2e', round(d['e2e']['value']))"
}
for i in $(seq $R); do
  for L in $LIBS; do PGB_LIBRARY=$PWD/$L one $L; done
  one in-tree
done
