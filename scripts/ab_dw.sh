set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
bash scripts/cifar_launches_env.sh dwdef
bash scripts/cifar_launches_env.sh dwtma PGB_TMA_ALL=1
for e in "" "PGB_TMA_ALL=1"; do env $e python bench.py --model cifar_cnn --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200; done
