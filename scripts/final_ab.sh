# Round-2 A/B evidence: MNIST throughput vs batch; CIFAR with each round-2 path switched off
for b in 256 512 1024 2048; do
  timeout 300 python bench.py --model mnist_cnn --batch $b --steps 300 --warmup 10 --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python -c "import json;d=json.load(open('/tmp/b.json'));print('mnist_cnn B=$b', round(d['value']), 'ex/s', d['kernels_us'])"
done
for v in "" PGB_NO_GHOST=1 PGB_NO_HALO=1 PGB_NO_KSPLIT=1 PGB_POOL_GENERIC=1 PGB_NO_TMA=1; do
  env $v timeout 300 python bench.py --model cifar_cnn --steps 60 --warmup 5 --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python -c "import json;d=json.load(open('/tmp/b.json'));print('cifar_cnn ${v:-default}', round(d['value']), 'ex/s')"
done
for v in "" PGB_NO_EMB_FORK=1 PGB_EMB_AGG_SCALAR=1; do
  env $v timeout 300 python bench.py --model embed --steps 300 --warmup 5 --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python -c "import json;d=json.load(open('/tmp/b.json'));print('embed ${v:-default}', round(d['value']), 'ex/s')"
done
