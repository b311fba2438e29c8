# quick GPU iteration: bf16 parity/stage tests (hang-protected), then the default bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stages.py -q -x ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -25 > gpurun_out/q_tests.txt
echo "tests rc=$?"; tail -25 gpurun_out/q_tests.txt
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/q_bench.json 2>gpurun_out/q_bench.err
echo "bench rc=$?"; tail -3 gpurun_out/q_bench.err
python -c "import json; d=json.load(open('gpurun_out/q_bench.json')); print(round(d['value']), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value'])); print({k:(round(v['ms_per_launch'],3), round(v.get('sfu_frac',0),3), round(v.get('hbm_frac',0),3)) for k,v in d['kernels'].items()})"
