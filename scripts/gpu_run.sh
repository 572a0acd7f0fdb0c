timeout 90 python -m pytest tests -m gpu -q -x --timeout 60 -k "linear" 2>&1 | tail -2
timeout 90 python scripts/quick_time.py
