cd $GRAFT_REPO_ROOT
for v in 0 1 2; do
TCL_MIXER_DIAG=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b16.json 2>/dev/null
python -c "
import json; j=json.load(open('gpurun_out/b16.json'))
print('DIAG=$v', 'mixer', round(j['kernels']['mixer']['ms_per_launch'],4))"
done
timeout 600 python scripts/measure_configs.py 2>&1 | tail -8
