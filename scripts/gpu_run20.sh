python -m pytest tests/test_gpu_kbac.py tests/test_gpu_parity.py tests/test_gpu_stages.py -x -q 2>&1 | tail -20
python scripts/next_rows_time.py
