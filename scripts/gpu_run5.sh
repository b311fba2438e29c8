cd $GRAFT_REPO_ROOT
export TCL_DEBUG_SYNC=1
timeout 300 python -m pytest tests/test_gpu_stages.py -x -q 2>&1 | grep -v "^\[tcl\]" | tail -5
export TCL_DEBUG_SYNC=0
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_v5.json 2> gpurun_out/bench_v5.err; tail -5 gpurun_out/bench_v5.err
python -c "
import json; j=json.load(open('gpurun_out/bench_v5.json'))
print(j['value'], j['ms_per_step'], j['e2e'])
for k,v in j['kernels'].items(): print(k, round(v['ms_per_launch'],3), v['launches'], round(v['share'],3), {kk: round(vv,3) for kk,vv in v.items() if kk in ('hbm_frac','tflops','sfu_frac','gbs')})
"
ncu --set full --import-source on --clock-control none -k regex:k_gemm_tc -s 3 -c 4 -o gpurun_out/prof_gemm_v5 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu5.err
