# Mixer phase split (TCL_MIXER_DIAG) + source-level ncu capture of the mixer.
cd $GRAFT_REPO_ROOT
for dg in 0 1 2 3; do
  echo "diag=$dg"; TCL_MIXER_DIAG=$dg timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print({k: round(v['ms_per_launch'],3) for k,v in d['kernels'].items()})"
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_mixer_fused -s 4 -c 1 -o gpurun_out/prof_r2b_mixer python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/
