cd $GRAFT_REPO_ROOT
for v in "TCL_MIXER_OCC=2" "TCL_MIXER_OCC=3" "TCL_MIXER=ws"; do
  echo "=== $v"
  env $v timeout 300 python -m pytest tests/test_gpu_stages.py tests/test_gpu_parity.py -x -q -k "bf16 or stage" 2>&1 | tail -2
  env $v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b7.json 2>/dev/null
  python -c "
import json; j=json.load(open('gpurun_out/b7.json'))
print(j['value'], j['ms_per_step'], 'mixer', j['kernels']['mixer']['ms_per_launch'], 'peaks', {k: (round(v/1e12,2) if isinstance(v,float) else v) for k,v in j['peaks'].items()})
"
done
