# Mixer: branch-free ZOH reset, full-chunk fast paths, halved conv weights; unroll variants.
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stages.py -m gpu -x -q 2>&1 | tail -3
TCL_MIXER_UNR=2 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stages.py -m gpu -x -q 2>&1 | tail -3
run() { echo "$*"; env "$@" timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], {k: round(v['ms_per_launch'],3) for k,v in d['kernels'].items() if k=='mixer'})"; }
run X=0
run TCL_MIXER_UNR=2
run TCL_MIXER_UNR=4
run TCL_MIXER_DIAG=1
run TCL_MIXER_DIAG=2
run TCL_MIXER_DIAG=2 TCL_MIXER_UNR=2
