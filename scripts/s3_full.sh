# Session-3: the whole GPU suite, then the quick bench lines (scripts/s3_quick.sh minus its parity file).
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -6
SKIP_PARITY=1 bash scripts/s3_quick.sh
