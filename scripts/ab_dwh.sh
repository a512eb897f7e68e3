python -m pytest tests -m gpu -x -q -k "cifar or switches or conv or tma or golden" 2>&1 | tail -2
for e in "" "PGB_TMA_SPLIT=1" "" "PGB_TMA_SPLIT=1"; do
  echo "== $e"; env $e python bench.py --model cifar_cnn --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-120
done
bash scripts/cifar_launches_env.sh dwh
