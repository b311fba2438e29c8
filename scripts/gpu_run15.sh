cd $GRAFT_REPO_ROOT
export TCL_DEBUG_SYNC=1
timeout 300 python -m pytest tests/test_gpu_stages.py -x -q 2>&1 | grep -v "^\[tcl\]" | tail -3
export TCL_DEBUG_SYNC=0
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for v in 0 1; do
TCL_NO_MCAST=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b15.json 2>gpurun_out/b15.err; tail -2 gpurun_out/b15.err
python -c "
import json; j=json.load(open('gpurun_out/b15.json'))
print('NO_MCAST=$v', round(j['value']), round(j['ms_per_step'],3), 'in_proj', round(j['kernels']['in_proj']['ms_per_launch'],4), j['kernels']['in_proj']['hbm_frac'])"
done
