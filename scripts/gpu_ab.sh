# A/B of mixer variants on one box: exp/libtcl_base.so (HEAD) vs the working tree, alternating.
cd $GRAFT_REPO_ROOT
run() { echo -n "$* :: "; env "$@" timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value']), {k: round(v['ms_per_launch'],3) for k,v in d['kernels'].items() if k in ('mixer','in_proj','out_proj')})"; }
for rep in 1 2; do
  run TCL_LIB=$PWD/exp/libtcl_base.so
  for v in "$@"; do run $v; done
done
