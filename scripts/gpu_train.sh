#!/bin/bash
# training-path GPU checks (f4): parity tests, each file bounded by its own timeout
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/train_smi.txt 2>&1
timeout -s KILL ${T:-900} python -m pytest tests/test_gpu_train.py -q -x ${K:+-k "$K"} -p no:cacheprovider > gpurun_out/train_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/train_tests.log
tail -30 gpurun_out/train_tests.log
