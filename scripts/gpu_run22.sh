python scripts/next_rows_time.py
