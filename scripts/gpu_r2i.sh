cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2i.json 2> gpurun_out/bench_r2i.err; tail -2 gpurun_out/bench_r2i.err; cat gpurun_out/bench_r2i.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gemm_tc -s 5 -c 1 -o gpurun_out/prof_r2i_inproj python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
