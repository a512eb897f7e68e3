#!/bin/bash
# One iteration: GPU suite, CIFAR bench, CIFAR step launch list.
OUT=gpurun_out/${1:-r02h_it}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
for i in 1 2; do
timeout 600 python bench.py --model cifar_cnn --steps 300 --warmup 5 --epochs 2 --no-cpu-baseline 2>$OUT/cifar.err | tail -1 > $OUT/cifar_$i.json
python -c "import json;d=json.load(open('$OUT/cifar_$i.json'));print('cifar', round(d['value']), 'e2e', round(d['e2e']['value']), 'us/step', round(d['ms_per_step']*1e3,1), 'direct_dw', d['kernels_us'].get('conv_dw_pex_direct'))" || tail -3 $OUT/cifar.err
done
