cd $GRAFT_REPO_ROOT
TCL_MCAST=2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stages.py -m gpu -x -q 2>&1 | tail -2
for r in 1 2; do for v in 0 2 1; do
 echo -n "mcast=$v :: "; TCL_MCAST=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value']), {k: round(v['ms_per_launch'],4) for k,v in d['kernels'].items() if k in ('in_proj','mixer')})"
done; done
