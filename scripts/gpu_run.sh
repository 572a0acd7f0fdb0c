timeout 600 python -m pytest tests -m gpu -q -x --timeout 200 -k "block or linear" 2>&1 | tail -2
for i in 1 2; do timeout 90 python scripts/quick_time.py 2>/dev/null | grep block; done
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_prep.csv python scripts/block_once.py 2 prep > /dev/null 2>&1
