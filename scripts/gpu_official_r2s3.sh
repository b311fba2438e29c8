# Round-2 final evidence (session 3 build): GPU tests, smoke, bench (N=1 default), reference arm,
# every config, long, accuracy (full-size `large`), launch list + per-kernel ncu captures (incl. the
# fp32 path's k_mixer_f32 / k_gemm_tf32 at rdu), compute-sanitizer memcheck / racecheck / synccheck.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
python bench.py > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err; tail -2 gpurun_out/bench_r2.err; cut -c1-300 gpurun_out/bench_r2.json
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference_r2.json 2>/dev/null; cut -c1-200 gpurun_out/bench_reference_r2.json
bash scripts/configs_gpu.sh
echo -n "== long 131072 :: "; timeout 900 python bench.py --config long --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null > gpurun_out/bench_long.json; python -c "import json; d=json.load(open('gpurun_out/bench_long.json')); print(round(d['value']), round(d['ms_per_step'],3), round(d['e2e']['value']))"
timeout 1500 python scripts/measure_configs.py --full-large 2>&1 | tail -8
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for k in k_scan k_inconv k_xdt k_gemm_ln; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 4 -c 1 -o gpurun_out/prof_r2_$k -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
for k in k_enc12 k_topk_radix k_pack k_pool_bf16; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 3 -c 1 -o gpurun_out/prof_r2_$k -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_head -s 2 -c 1 -o gpurun_out/prof_r2_k_head -f python bench.py --config paper --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
# fp32 path at rdu (batched MC): the 3xTF32 in_proj (4th tf32 launch) and the fp32 mixer
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gemm_tf32 -s 3 -c 1 -o gpurun_out/prof_r2_k_gemm_tf32 -f python bench.py --config rdu --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_mixer_f32 -c 1 -o gpurun_out/prof_r2_k_mixer_f32 -f python bench.py --config rdu --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out/prof_r2_*
mkdir -p gpurun_out/sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 --log-file gpurun_out/sanitizer/$tool.log \
      python scripts/sanitize_run.py > gpurun_out/sanitizer/$tool.out 2>&1
  echo "== $tool rc=$? :: $(tail -1 gpurun_out/sanitizer/$tool.out) :: $(tail -1 gpurun_out/sanitizer/$tool.log)"
done
