cd $GRAFT_REPO_ROOT
TCL_MIXER_DIAG=0 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('mixer', j['kernels']['mixer']['ms_per_launch'])"
TCL_MIXER_DIAG=4 timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep "mixer diag" | tail -6
