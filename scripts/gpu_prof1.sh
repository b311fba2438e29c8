cd $GRAFT_REPO_ROOT
ncu --set full --import-source on --clock-control none -k regex:k_mixer_fused -s 2 -c 1 -o gpurun_out/prof_mixer_v2 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu1.err
ncu --set full --import-source on --clock-control none -k regex:k_gemm_tc -s 5 -c 3 -o gpurun_out/prof_gemm_v2 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu2.err
ncu --set full --import-source on --clock-control none -k regex:k_head -s 1 -c 1 -o gpurun_out/prof_head_v2 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu3.err
ls -la gpurun_out/
