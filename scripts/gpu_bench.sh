# bench + ncu evidence on one B200 (run under gpurun from the repo root)
set -x
mkdir -p gpurun_out
timeout 600 python bench.py 2>gpurun_out/bench.err | tee gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fmha_bf16 -s 4 -c 2 -o gpurun_out/prof_fmha -f \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_fmha.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 12 -c 4 -o gpurun_out/prof_gemm -f \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_gemm.log 2>&1
ls -la gpurun_out
