#!/bin/bash
# training step bench (f4) + ncu launch list of the same command (per-kernel shares)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -s KILL 300 python bench.py --config train --steps 20 --warmup 5 > gpurun_out/train_bench.json 2> gpurun_out/train_bench.err
echo "bench rc=$?"; cat gpurun_out/train_bench.json; tail -3 gpurun_out/train_bench.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file gpurun_out/train_launches.csv python bench.py --config train --steps 1 --warmup 3 > gpurun_out/train_ncu.log 2>&1
echo "ncu rc=$?"
