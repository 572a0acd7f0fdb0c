#!/bin/bash
# A/B of the attention-backward item walk (DSP_FMHA_BWD_CH) on one box, plus its parity tests per walk
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do for ch in 1 2 4 8 0; do
  DSP_FMHA_BWD_CH=$ch timeout -s KILL 120 python scripts/fmha_bwd_walk_ab.py 2>&1 | tail -1
done; done | tee gpurun_out/fmha_bwd_walk_ab.txt
for ch in 0 4; do
  DSP_FMHA_BWD_CH=$ch timeout -s KILL 300 python -m pytest tests/test_gpu_train.py -q -x -k "attention" -p no:cacheprovider 2>&1 | tail -1
done
