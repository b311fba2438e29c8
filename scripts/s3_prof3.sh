# Session-3: parity (incl. the d_model 240 fp32 case), then ncu of the 3xTF32 GEMMs at rdu after the epilogue change.
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tf32 -c 5 -o gpurun_out/s3_tf32b -f \
  python bench.py --config rdu --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/s3_tf32b.log 2>&1
ls gpurun_out | tail -3
