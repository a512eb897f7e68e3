#!/bin/bash
# Final evidence of this session: GPU suite, smoke, per-config bench lines, driver-setting bench
# of both arms, CIFAR launch list.
OUT=gpurun_out/r02h_final; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
bash scripts/bench_all.sh r02h_all 300 > $OUT/configs.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
bash scripts/cifar_launches_env.sh r02h_final_cifar
tail -2 $OUT/pytest_gpu.log; cat $OUT/smoke.log; cat $OUT/configs.txt | cut -c1-200
