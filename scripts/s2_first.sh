cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/s2_gputests.txt
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s2_bench.json 2>gpurun_out/s2_bench.err
tail -3 gpurun_out/s2_gputests.txt
python -c "import json; d=json.load(open('gpurun_out/s2_bench.json')); print(round(d['value']), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value'])); print({k:(round(v['ms_per_launch'],3), round(v.get('sfu_frac',0),3), round(v.get('hbm_frac',0),3)) for k,v in d['kernels'].items()})"
