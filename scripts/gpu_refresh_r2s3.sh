# Refresh after the last session-3 changes (Philox inlined, LN fusion at d_model <= 128, NVTX /
# NCCL async-error, k_scan dynamic work groups, 20-warp k_xdt): default bench line, every config, launch list (same files as gpu_official_r2s3.sh).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err; tail -1 gpurun_out/bench_r2.err; cut -c1-200 gpurun_out/bench_r2.json
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference_r2.json 2>/dev/null; cut -c1-120 gpurun_out/bench_reference_r2.json
bash scripts/configs_gpu.sh
echo -n "== long 131072 :: "; timeout 900 python bench.py --config long --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null > gpurun_out/bench_long.json; python -c "import json; d=json.load(open('gpurun_out/bench_long.json')); print(round(d['value']), round(d['ms_per_step'],3), round(d['e2e']['value']))"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_scan -s 4 -c 1 -o gpurun_out/prof_r2_k_scan -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_xdt -s 4 -c 1 -o gpurun_out/prof_r2_k_xdt -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gemm_tf32 -s 3 -c 1 -o gpurun_out/prof_r2_k_gemm_tf32 -f python bench.py --config rdu --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_mixer_f32 -c 1 -o gpurun_out/prof_r2_k_mixer_f32 -f python bench.py --config rdu --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out | wc -l
