cd $GRAFT_REPO_ROOT
ncu --set full --import-source on --clock-control none -k regex:k_mixer_fused -s 1 -c 1 -o gpurun_out/prof_mixer_fused_v8 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu8a.err
TCL_MIXER=ws ncu --set full --import-source on --clock-control none -k regex:k_mixer_ws -s 1 -c 1 -o gpurun_out/prof_mixer_ws_v8 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu8b.err
TCL_MIXER=ws timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b8.json 2>/dev/null
python -c "
import json; j=json.load(open('gpurun_out/b8.json'))
print('ws OFF=0', j['value'], j['ms_per_step'], 'mixer', j['kernels']['mixer']['ms_per_launch'])"
