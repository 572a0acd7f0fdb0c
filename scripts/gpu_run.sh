set -x
timeout 300 python -m pytest tests -m gpu -q -x --timeout 120 -k "linear" 2>&1 | tail -15
timeout 300 python scripts/quick_time.py
timeout 900 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -8
