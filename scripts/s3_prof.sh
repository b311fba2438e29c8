# Session-3 ncu captures: the large-batch decoder launch (k_head, pooled_ready) and the 3xTF32 GEMMs at rdu.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_head -c 1 -o gpurun_out/s3_head -f \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/s3_head.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tf32 -c 5 -o gpurun_out/s3_tf32 -f \
  python bench.py --config rdu --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/s3_tf32.log 2>&1
ls -la gpurun_out
