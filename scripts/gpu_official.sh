# Final round-1 evidence: GPU tests, smoke, bench (N=1, default), reference arm, every config,
# launch list + per-kernel ncu captures.
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
python bench.py > gpurun_out/bench_official.json 2> gpurun_out/bench_official.err; tail -2 gpurun_out/bench_official.err
cat gpurun_out/bench_official.json
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference.json 2>/dev/null; cat gpurun_out/bench_reference.json
for c in tiny tuning rdu paper; do for pr in fp32 bf16; do
  echo -n "== $c $pr :: "; timeout 600 python bench.py --config $c --precision $pr --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null > gpurun_out/bench_${c}_${pr}.json; python -c "import json,sys; d=json.load(open('gpurun_out/bench_${c}_${pr}.json')); print(round(d['value']), round(d['ms_per_step'],4), round(d['e2e']['value']), d['roofline']['kernel'], round(d['roofline']['frac'],3))"
done; done
echo -n "== long 131072 :: "; timeout 900 python bench.py --config long --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null > gpurun_out/bench_long.json; python -c "import json; d=json.load(open('gpurun_out/bench_long.json')); print(round(d['value']), round(d['ms_per_step'],3), round(d['e2e']['value']))"
timeout 900 python scripts/measure_configs.py 2>&1 | tail -8
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_official.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for k in k_mixer_fused k_gemm_tc k_gemm_ln k_gemm_simt; do
  ncu --set full --import-source on --clock-control none -k regex:$k -s 4 -c 1 -o gpurun_out/prof_official_$k python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:k_enc12 -s 3 -c 1 -o gpurun_out/prof_official_k_enc12 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_topk_radix -s 3 -c 1 -o gpurun_out/prof_official_k_topk_radix python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_pack -s 3 -c 1 -o gpurun_out/prof_official_k_pack python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_pool -s 3 -c 1 -o gpurun_out/prof_official_k_pool_bf16 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out/prof_official_*
