cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stages.py -m gpu -x -q 2>&1 | tail -3
TCL_MIXER=pp timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stages.py -m gpu -x -q 2>&1 | tail -3
bash scripts/gpu_ab.sh X=0 TCL_MIXER=pp
