cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_v4.json 2> gpurun_out/bench_v4.err; tail -5 gpurun_out/bench_v4.err
python -c "
import json; j=json.load(open('gpurun_out/bench_v4.json'))
print(j['value'], j['ms_per_step'], j['e2e'])
for k,v in j['kernels'].items(): print(k, round(v['ms_per_launch'],3), v['launches'], round(v['share'],3), {kk: round(vv,3) for kk,vv in v.items() if kk in ('hbm_frac','tflops','sfu_frac','gbs')})
"
ncu --set full --import-source on --clock-control none -k regex:k_mixer_fused -s 1 -c 1 -o gpurun_out/prof_mixer_v4 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu4.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
