# Throughput of every BASELINE.json configuration on one GPU (bench.py per config) + accuracy table.
cd $GRAFT_REPO_ROOT
for c in tiny tuning rdu paper large; do
  echo "== $c"; timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(json.dumps({k: d[k] for k in ('value','ms_per_step','e2e','gpu_launches')}), json.dumps({k: round(v['ms_per_launch'],4) for k,v in d['kernels'].items()}))"
done
echo "== long (131072 per GPU)"; timeout 900 python bench.py --config long --n 131072 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(json.dumps({k: d[k] for k in ('value','ms_per_step','e2e')}), json.dumps({k: round(v['ms_per_launch'],4) for k,v in d['kernels'].items()}))"
timeout 900 python scripts/measure_configs.py 2>&1 | tail -20
