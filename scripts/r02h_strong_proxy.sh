#!/bin/bash
# Per-rank cost of the strong-scaling split on one GPU: global batch 256 over N ranks
# means B = 256 / N per rank; --dist-schedule runs the multi-GPU kernels (aggregate mode 1,
# one-rank NCCL all-reduce, noise_update) so only the NVLink transfer itself is missing.
OUT=gpurun_out/${1:-r02h_proxy}; mkdir -p $OUT
for M in mnist_cnn cifar_cnn; do
  for Bt in 32 64 128 256; do
    for D in "" "--dist-schedule"; do
      S=2000; [ $M = cifar_cnn ] && S=100
      tag=${M}_${Bt}${D:+_dist}
      timeout 600 python bench.py --model $M --batch $Bt $D --steps $S --warmup 10 --epochs 2 --no-cpu-baseline > $OUT/$tag.json 2> $OUT/$tag.err
      python -c "import json;d=json.load(open('$OUT/$tag.json'));print('$tag', 'value', round(d['value']), 'us/step', round(d['ms_per_step']*1e3,2), 'e2e', round(d['e2e']['value']), d['kernels_us'])" || tail -3 $OUT/$tag.err
    done
  done
done
