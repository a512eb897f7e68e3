# MNIST long-run A/B on one box: the current tree vs an older build staged in _old/
for i in 1 2; do
  python bench.py --steps 2000 --warmup 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('cur',d['value'],d['ms_per_step'])"
  (cd _old && python bench.py --steps 2000 --warmup 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('old',d['value'],d['ms_per_step'])")
done
