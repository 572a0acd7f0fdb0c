timeout 300 python -m pytest tests -m gpu -q -x --timeout 120 -k "layer_norm or block_bf16_full" 2>&1 | tail -2
timeout 90 python scripts/quick_time.py | grep -E "block|layernorm"
DSP_FOLD_LN=1 timeout 90 python scripts/quick_time.py | grep -E "block"
timeout 300 python bench.py --steps 20 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step']); [print(k, v) for k,v in d['stages'].items()]"
