cd $GRAFT_REPO_ROOT
for off in 0 1 2; do
  TCL_MIXER_OFF=$off timeout 300 python -m pytest tests/test_gpu_stages.py -x -q -k "large-1" 2>&1 | tail -1
  for rep in 1 2; do
  TCL_MIXER_OFF=$off timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b14.json 2>/dev/null
  python -c "
import json; j=json.load(open('gpurun_out/b14.json'))
print('OFF=$off', round(j['value']), round(j['ms_per_step'],3), 'mixer', round(j['kernels']['mixer']['ms_per_launch'],3))"
  done
done
