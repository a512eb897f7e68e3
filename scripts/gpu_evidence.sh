#!/bin/bash
# Round evidence for the MNIST headline: GPU tests, smoke, bench (default
# flags), ncu launch list, one ncu --set full capture of the step kernels and
# the device phase trace. Usage: bash scripts/gpu_evidence.sh <tag>
TAG=${1:-ev}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 200 --csv \
   --log-file $OUT/launches.csv python bench.py --steps 30 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:tc_kernel|aggregate_kernel" -s 10 -c 2 \
   -o $OUT/prof python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/ncu_full.log 2>&1
PGB_TRACE=1 python paper_2010_09063_b200/build.py > /dev/null 2>&1
timeout 300 python scripts/trace_phases.py > $OUT/trace.txt 2>&1
timeout 300 python scripts/trace_phases.py --graph > $OUT/trace_graph.txt 2>&1
for f in $OUT/*.log; do tail -n 2 $f; done
cat $OUT/bench.json
