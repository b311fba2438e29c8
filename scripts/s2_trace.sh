cd $GRAFT_REPO_ROOT
python exp/inconv_trace.py large 2>&1 | tail -20
