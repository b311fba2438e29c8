cd $GRAFT_REPO_ROOT
for c in tuning rdu paper; do for pr in fp32 bf16; do
  echo -n "== $c $pr :: "; timeout 600 python bench.py --config $c --precision $pr --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value']), round(d['ms_per_step'],4), round(d['e2e']['value']), json.dumps({k: round(v['ms_per_launch'],4) for k,v in d['kernels'].items()}))"
done; done
