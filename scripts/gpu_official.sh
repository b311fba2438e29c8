# GPU tests, one full bench line (N=1, default config) + the ncu evidence kept under profiles/.
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
python bench.py > gpurun_out/bench_official.json 2> gpurun_out/bench_official.err; tail -2 gpurun_out/bench_official.err
cat gpurun_out/bench_official.json
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference.json 2>/dev/null; cat gpurun_out/bench_reference.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_official.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for k in k_mixer_fused k_gemm_tc k_gemm_ln k_pool_bf16 k_pack k_topk_chunk k_gemm_simt; do
  ncu --set full --import-source on --clock-control none -k regex:$k -s 4 -c 1 -o gpurun_out/prof_official_$k python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
ls gpurun_out/prof_official_*
