# Session-3 quick GPU iteration: parity file (unless SKIP_PARITY), then bench lines.
cd $GRAFT_REPO_ROOT
[ -z "$SKIP_PARITY" ] && timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stages.py -q -x 2>&1 | tail -4
b() { python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['config'], d['config'].get('precision'), round(d['value']), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value'])); print({k:(round(v['ms_per_launch'],3), round(v.get('hbm_frac',0),3)) for k,v in d['kernels'].items()})"; }
for c in ${CONFIGS:-large rdu tuning}; do b --config $c; done
if [ -f exp/libtcl_ab.so ]; then echo "== A/B: exp/libtcl_ab.so"; TCL_LIB=exp/libtcl_ab.so b --config ${AB_CONFIG:-large}; fi
