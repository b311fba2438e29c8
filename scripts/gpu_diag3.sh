cd $GRAFT_REPO_ROOT
for v in 0 3 2 1; do
TCL_MIXER_DIAG=$v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('diag $v mixer', j['kernels']['mixer']['ms_per_launch'])"
done
