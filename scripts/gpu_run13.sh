cd $GRAFT_REPO_ROOT
export TCL_DEBUG_SYNC=1
timeout 300 python -m pytest tests/test_gpu_stages.py -x -q -s 2>&1 | grep -v "^\[tcl\]" | tail -6
export TCL_DEBUG_SYNC=0
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -8
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b13.json 2>gpurun_out/b13.err; tail -3 gpurun_out/b13.err
python -c "
import json; j=json.load(open('gpurun_out/b13.json'))
print(j['value'], j['ms_per_step'])
for k,v in j['kernels'].items(): print(k, round(v['ms_per_launch'],3), v['launches'], round(v['share'],3), {kk: round(vv,3) for kk,vv in v.items() if kk in ('hbm_frac','tflops','sfu_frac','gbs')})
"
timeout 600 python bench.py --config long --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b13_long.json 2>gpurun_out/b13_long.err; tail -3 gpurun_out/b13_long.err
python -c "
import json; j=json.load(open('gpurun_out/b13_long.json'))
print('long', j['value'], j['ms_per_step'], j['config'])"
