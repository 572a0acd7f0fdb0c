# Round evidence on one B200 (run under gpurun from the repo root):
#   bench JSON, ncu launch list of the same bench command, ncu --set full of the top kernels.
set -x
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fmha -s 2 -c 2 -o gpurun_out/prof_fmha -f \
   python scripts/prof_kernels.py fmha > gpurun_out/ncu_fmha.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm -s 2 -c 2 -o gpurun_out/prof_gemm -f \
   python scripts/prof_kernels.py gemm > gpurun_out/ncu_gemm.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:layer_norm -s 1 -c 1 -o gpurun_out/prof_ln -f \
   python scripts/prof_kernels.py ln > gpurun_out/ncu_ln.log 2>&1
ls -la gpurun_out
