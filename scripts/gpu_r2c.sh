# Mixer experiments: scan unroll, CTA stagger.
cd $GRAFT_REPO_ROOT
run() { echo "$*"; env "$@" timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], {k: round(v['ms_per_launch'],3) for k,v in d['kernels'].items() if k=='mixer'})"; }
run X=0
run TCL_MIXER_UNR=2
for st in 3000 6000 9000 12000 18000; do run TCL_MIXER_STAGGER=$st; done
run TCL_MIXER_UNR=2 TCL_MIXER_STAGGER=9000
run TCL_MIXER_DIAG=2 TCL_MIXER_UNR=2
