timeout 200 python -m pytest tests -m gpu -q -x --timeout 100 -k "attention_core or stage or long or block_bf16" 2>&1 | tail -1
for i in 1 2; do
timeout 90 python scripts/quick_time.py | grep -E "block|fmha t"
DSP_LIB_OVERRIDE=$PWD/paper_2403_10266_b200/libdsp_old.so timeout 90 python scripts/quick_time.py | grep -E "block|fmha t" | sed 's/^/OLD /'
done
