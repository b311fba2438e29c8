python -m pytest tests/test_gpu_train.py -x -q 2>&1 | tail -5
python scripts/next_rows_time.py 2>&1 | tail -2
