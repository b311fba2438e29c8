python -m pytest tests/test_gpu_topk_score.py tests/test_gpu_rdu.py -x -q 2>&1 | tail -20
python scripts/rdu_time.py
