# full GPU suite (hang-protected) + the default bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/f_tests.txt
echo "tests rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/f_tests.txt | tail -8
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/q_bench.json 2>gpurun_out/q_bench.err
echo "bench rc=$?"; tail -3 gpurun_out/q_bench.err
python -c "import json; d=json.load(open('gpurun_out/q_bench.json')); print(round(d['value']), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value'])); print({k:(round(v['ms_per_launch'],3), round(v.get('hbm_frac',0),3)) for k,v in d['kernels'].items()})"
