# FCNN / logreg / embed throughput vs mlp::kWarps (examples per CTA of mlp_kernel)
for w in 8 4 2; do
  sed -i "s/^constexpr int kWarps = [0-9]*;  \/\/ examples per CTA/constexpr int kWarps = $w;  \/\/ examples per CTA/" paper_2010_09063_b200/csrc/mlp_fused.cuh
  python paper_2010_09063_b200/build.py > /dev/null 2>&1 || { echo build failed; exit 1; }
  for M in fcnn logreg embed; do
    timeout 300 python bench.py --model $M --steps 300 --warmup 5 --no-cpu-baseline > /tmp/b.json 2>/dev/null
    python -c "import json;d=json.load(open('/tmp/b.json'));print('kWarps $w', '$M', round(d['value']), d['kernels_us'])"
  done
done
