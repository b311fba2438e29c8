cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "topk" 2>&1 | tail -2
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gemm_simt128 -s 6 -c 1 -o gpurun_out/prof_r3b_simt128 python bench.py --config rdu --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out/prof_r3b*
