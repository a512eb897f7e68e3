#!/bin/bash
# ncu evidence for every BASELINE config's step kernels:
# per config, a launch list (gpu__time_duration, clocks not locked) and one
# ncu --set full capture of each distinct step kernel (with source), plus the
# MNIST device phase traces. Usage: bash scripts/gpu_profile_all.sh <tag>
TAG=${1:-prof}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python paper_2010_09063_b200/build.py > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
for M in mnist_cnn cifar_cnn fcnn logreg embed; do
  S=30; [ $M = cifar_cnn ] && S=6
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 300 --csv \
     --log-file $OUT/launches_$M.csv python bench.py --model $M --steps $S --warmup 3 --epochs 1 \
     --no-cpu-baseline > $OUT/ncu_launch_$M.log 2>&1
  # one full capture per distinct kernel of the step: skip the warm-up launches
  timeout 1500 ncu --set full --clock-control none --import-source on -s 60 -c 24 \
     -o $OUT/full_$M python bench.py --model $M --steps 4 --warmup 3 --epochs 1 \
     --no-cpu-baseline > $OUT/ncu_full_$M.log 2>&1
  python scripts/ncu_summary.py $OUT/full_$M.ncu-rep 16 > $OUT/summary_$M.txt 2>&1
  python scripts/ncu_traffic_json.py $OUT/full_$M.ncu-rep $OUT/traffic_$M.json "$TAG $M ncu --set full" > /dev/null 2>&1
  # reports with source are tens of MB: keep them only when small (gpurun_out <= 64 MiB)
  [ $(stat -c %s $OUT/full_$M.ncu-rep 2>/dev/null || echo 0) -gt 12000000 ] && rm -f $OUT/full_$M.ncu-rep
done
PGB_TRACE=1 python paper_2010_09063_b200/build.py > /dev/null 2>&1
timeout 300 python scripts/trace_phases.py > $OUT/trace.txt 2>&1
timeout 300 python scripts/trace_phases.py --graph > $OUT/trace_graph.txt 2>&1
ls -la $OUT
