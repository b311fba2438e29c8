cd $GRAFT_REPO_ROOT
for v in 0 1 2 3; do
TCL_MIXER_VAR=$v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('var $v mixer', j['kernels']['mixer']['ms_per_launch'], 'value', j['value'])"
done
TCL_MIXER_VAR=3 python -m pytest tests/test_gpu_parity.py -q -x -k "bf16 or large" 2>&1 | tail -2
