mkdir -p gpurun_out/dwh
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:tma_dw_halo" -s 3 -c 3 \
   -o gpurun_out/dwh/prof python bench.py --model cifar_cnn --steps 6 --warmup 3 --epochs 1 --no-cpu-baseline > gpurun_out/dwh/ncu.log 2>&1
tail -3 gpurun_out/dwh/ncu.log
