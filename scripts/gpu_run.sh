timeout 300 python -m pytest tests/test_gpu_block.py -m gpu -q -x --timeout 120 -k "virtual" 2>&1 | tail -3
