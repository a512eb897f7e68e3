bash scripts/gpu_quick.sh q12
PGB_NO_PDL=1 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline > gpurun_out/q12/nopdl.json; python -c "import json;d=json.load(open('gpurun_out/q12/nopdl.json'));print('nopdl',d['value'],d['e2e']['value'])"
python scripts/trace_phases.py
