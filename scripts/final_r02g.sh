bash scripts/gpu_round.sh r02g > gpurun_out/r02g_round.txt 2>&1
bash scripts/bench_all.sh r02g_all 300 > gpurun_out/r02g_configs.txt 2>&1
bash scripts/cifar_launches_env.sh r02g_cifar
bash scripts/gpu_prof.sh r02g_prof cifar_cnn "tma_dw_halo|tma_gemm_kernel|conv3x3_smallc" > gpurun_out/r02g_prof.txt 2>&1
