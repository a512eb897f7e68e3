for cfg in "4 4" "8 4" "4 8" "2 2"; do
  set -- $cfg
  echo "== fwd $1 dx $2"
  PGB_KSPLIT_CHAIN_FWD=$1 PGB_KSPLIT_CHAIN_DX=$2 TAG="f$1d$2" timeout 200 python scripts/golden_cifar_dbg.py | awk '{print $2, $5, $7, $8}' | tr '\n' ' '; echo
  PGB_KSPLIT_CHAIN_FWD=$1 PGB_KSPLIT_CHAIN_DX=$2 timeout 300 python bench.py --model cifar_cnn --steps 60 --warmup 5 --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python -c "import json;d=json.load(open('/tmp/b.json'));print('value', d['value'])"
done
