cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for pr in fp32 bf16; do
  echo -n "== rdu $pr :: "; timeout 600 python bench.py --config rdu --precision $pr --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value']), round(d['ms_per_step'],4), round(d['e2e']['value']), json.dumps({k: round(v['ms_per_launch'],4) for k,v in d['kernels'].items()}))"
done
