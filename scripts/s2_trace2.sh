cd $GRAFT_REPO_ROOT
bash exp/trace_build.sh > /dev/null 2>&1
python exp/inmix_trace.py large 2>&1 | sed -n 1,14p
EXTRA_DEFS=-DTCL_INMIX_NOSTORE bash exp/trace_build.sh > /dev/null 2>&1
echo NOSTORE; python exp/inmix_trace.py large 2>&1 | sed -n 1,14p
