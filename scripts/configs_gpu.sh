# Every configuration's bench line (value, ms/step, e2e, dominant kernel + fraction).
cd $GRAFT_REPO_ROOT
for c in tiny tuning rdu paper; do for pr in fp32 bf16; do
  echo -n "== $c $pr :: "; timeout 600 python bench.py --config $c --precision $pr --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null > gpurun_out/bench_${c}_${pr}.json; python -c "import json,sys; d=json.load(open('gpurun_out/bench_${c}_${pr}.json')); print(round(d['value']), round(d['ms_per_step'],4), round(d['e2e']['value']), d['roofline']['kernel'], round(d['roofline']['frac'],3), d['gpu_launches'])"
done; done
