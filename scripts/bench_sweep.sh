#!/bin/bash
# BASELINE config 2: FFNN batch sweep (16-512), our arm and the reference arm per batch.
OUT=gpurun_out/${1:-sweep}; mkdir -p $OUT
for Bt in 16 32 64 128 256 512; do
  timeout 300 python bench.py --model fcnn --batch $Bt --steps ${2:-500} --warmup 5 --no-cpu-baseline > $OUT/fcnn_$Bt.json 2> $OUT/fcnn_$Bt.err
  timeout 300 python bench.py --model fcnn --batch $Bt --impl reference --steps 20 --warmup 2 --ref-seconds 5 > $OUT/fcnn_ref_$Bt.json 2> $OUT/fcnn_ref_$Bt.err
  python -c "import json;d=json.load(open('$OUT/fcnn_$Bt.json'));r=json.load(open('$OUT/fcnn_ref_$Bt.json'));print('fcnn B=$Bt', round(d['value']), 'e2e', round(d['e2e']['value']), 'reference', round(r['value']))" || tail -3 $OUT/fcnn_$Bt.err
done
