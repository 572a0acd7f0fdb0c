set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import torch;print(torch.cuda.get_device_name())"
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "linear or layer_norm" 2>&1 | tail -30
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "attention_core" 2>&1 | tail -30
