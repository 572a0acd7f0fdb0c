#!/bin/bash
# ncu --set full of the training step's attention-backward and LayerNorm-backward kernels
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -s KILL 300 python bench.py --config train --steps 10 --warmup 3 > gpurun_out/train_bench.json 2> gpurun_out/train_bench.err
echo "bench rc=$?"; cat gpurun_out/train_bench.json
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"fmha_bwd|ln_bwd_bf16|ln_bwd_param" \
  --launch-skip ${SKIP:-0} -c ${COUNT:-6} -o gpurun_out/train_prof -f python bench.py --config train --steps 1 --warmup 3 > gpurun_out/train_prof.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/train_prof.log
