# CIFAR bench A/B over env settings given as arguments ("" = default)
for e in "$@"; do
  echo "== $e"; env $e python bench.py --model cifar_cnn --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-120
done
