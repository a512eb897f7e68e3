for c in 1 2 4; do
  PGB_KSPLIT_CHAIN=$c TAG=c$c timeout 200 python scripts/golden_cifar_dbg.py | awk '{print $2, $8, $9}' | tr '\n' ' '; echo
  PGB_KSPLIT_CHAIN=$c timeout 300 python bench.py --model cifar_cnn --steps 60 --warmup 5 --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python -c "import json;d=json.load(open('/tmp/b.json'));print('chain $c value', d['value'], d['kernels_us']['conv_fwd_tma'], d['kernels_us']['conv_bwd_x_tma'], d['kernels_us']['conv_dw_sum'])"
done
