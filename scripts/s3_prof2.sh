# Session-3 ncu capture of the fp32 mixer at rdu (batched MC).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mixer_f32 -c 1 -o gpurun_out/s3_mixf32 -f \
  python bench.py --config rdu --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/s3_mixf32.log 2>&1
ls -la gpurun_out | tail -3
