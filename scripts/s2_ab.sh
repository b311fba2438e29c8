# A/B: the default build vs exp/libtcl_ab.so (bench twice each, alternating) + bf16 parity with B
cd $GRAFT_REPO_ROOT
for r in 1 2; do
  for v in A B; do
    if [ $v = B ]; then export TCL_LIB=$GRAFT_REPO_ROOT/exp/libtcl_ab.so; else unset TCL_LIB; fi
    timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null > gpurun_out/ab_$v.json
    python -c "import json; d=json.load(open('gpurun_out/ab_$v.json')); print('$v', round(d['ms_per_step'],3), {k:round(v['ms_per_launch'],3) for k,v in d['kernels'].items() if k in ('scan','in_proj','xdt','out_proj')})"
  done
done
export TCL_LIB=$GRAFT_REPO_ROOT/exp/libtcl_ab.so
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -2
