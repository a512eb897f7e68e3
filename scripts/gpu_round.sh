#!/bin/bash
# GPU iteration: full GPU test suite (no -x: every failure listed), the
# driver-setting bench (--steps 20 --warmup 5) and a long bench.
# Usage: bash scripts/gpu_round.sh <tag> [pytest -k expr]
TAG=${1:-r}; K=${2:-}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python paper_2010_09063_b200/build.py > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
if [ -n "$K" ]; then timeout 1500 python -m pytest tests -m gpu -q -k "$K" -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1
else timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; fi
echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -n 30 $OUT/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench_driver.json 2> $OUT/bench_driver.err
tail -n 3 $OUT/bench_driver.err
timeout 600 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline > $OUT/bench_long.json 2> $OUT/bench_long.err
tail -n 3 $OUT/bench_long.err
for f in bench_driver bench_long; do
python -c "import json;d=json.load(open('$OUT/$f.json'));print('$f value',d['value'],'e2e',d['e2e']['value'],'epoch_s',d['e2e']['median_epoch_s'],'host_issue',d['host_issue_us_per_step'],'kernels_us',d['kernels_us'])"
done
