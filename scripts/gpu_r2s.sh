cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
run() { echo -n "$* :: "; env "$@" timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value']), {k: round(v['ms_per_launch'],3) for k,v in d['kernels'].items()})"; }
for r in 1 2; do run TCL_ENC12=0; run TCL_ENC12=1; run TCL_LIB=$PWD/exp/libtcl_base.so TCL_ENC12=0; done
