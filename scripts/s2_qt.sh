# quick: bf16 parity + stage tests, bench, inconv trace
cd $GRAFT_REPO_ROOT
bash scripts/s2_quick.sh
python exp/inconv_trace.py large 2>&1 | tail -9
