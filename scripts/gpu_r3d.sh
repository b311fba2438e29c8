cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for f in 0 1; do for c in tuning rdu paper; do
  echo -n "== $c FUSE_LN=$f :: "; TCL_F32_FUSE_LN=$f timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value']), round(d['ms_per_step'],4), json.dumps({k: round(v['ms_per_launch'],4) for k,v in d['kernels'].items()}))"
done; done
