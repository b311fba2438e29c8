python -m pytest tests/test_gpu_rdu.py -x -q 2>&1 | tail -15
python scripts/next_rows_time.py 2>&1 | head -4
