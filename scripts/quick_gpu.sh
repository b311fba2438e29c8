# Quick GPU iteration: bf16 parity + stage tests, then the default bench line's per-kernel times.
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stages.py -q -x -s ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | grep -E "FAIL|Error|error|passed|failed|spearman|Assert|prec " | tail -30
python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value'])); print({k:(round(v['ms_per_launch'],3), round(v.get('sfu_frac',0),3), round(v.get('hbm_frac',0),3)) for k,v in d['kernels'].items()})"
