mkdir -p gpurun_out/fwd
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:tma_gemm_kernel" -s 0 -c 1 \
   -o gpurun_out/fwd/prof python bench.py --model cifar_cnn --steps 4 --warmup 3 --epochs 1 --no-cpu-baseline > gpurun_out/fwd/ncu.log 2>&1
tail -2 gpurun_out/fwd/ncu.log
