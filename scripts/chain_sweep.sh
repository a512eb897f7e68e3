for c in 4 8 16 1000; do
  PGB_KSPLIT_CHAIN=$c timeout 300 python bench.py --model cifar_cnn --steps 60 --warmup 5 --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python -c "import json;d=json.load(open('/tmp/b.json'));print('chain', $c, d['value'])"
done
