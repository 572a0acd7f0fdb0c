# Round-2 final evidence at the last HEAD: GPU suite (-rP margins), smoke, bench lines, reference arm,
# ncu launch lists (forward, training step), ncu --set full of the attention backward and a wgrad GEMM
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1700 python -m pytest tests -m gpu -q -rP -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cut -c1-200 gpurun_out/bench.json
timeout 600 python bench.py --config long --steps 5 > gpurun_out/bench_long.json 2>&1; cut -c1-200 gpurun_out/bench_long.json
timeout 600 python bench.py --config model28 --steps 5 > gpurun_out/bench_model28.json 2>&1; cut -c1-200 gpurun_out/bench_model28.json
timeout 600 python bench.py --config train --steps 30 > gpurun_out/bench_train.json 2>&1; cut -c1-200 gpurun_out/bench_train.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2>&1; cut -c1-200 gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/train_launches.csv \
   python bench.py --config train --steps 1 --warmup 3 > gpurun_out/train_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fmha_bwd -s 1 -c 1 -o gpurun_out/prof_fmha_bwd -f \
   python bench.py --config train --steps 1 --warmup 3 > gpurun_out/ncu_fmha_bwd.log 2>&1
ls -la gpurun_out
