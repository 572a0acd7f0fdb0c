# T=128 single-tile FMHA kernel: parity tests, A/B timing, ncu, long bench
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_edge.py tests/test_gpu_configs.py -q -x --timeout 400 -k "attention or attn or ragged or long or cross" > gpurun_out/pytest_fmha.log 2>&1; tail -3 gpurun_out/pytest_fmha.log
for v in "" noseq; do
  if [ -z "$v" ]; then timeout 120 python scripts/fmha_time.py; else DSP_LIB_OVERRIDE=paper_2403_10266_b200/libdsp_$v.so timeout 120 python scripts/fmha_time.py; fi
done > gpurun_out/fmha_ab.txt 2>&1; grep spatial gpurun_out/fmha_ab.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fmha -s 2 -c 1 -o gpurun_out/prof_fmha_tlong -f \
   python scripts/prof_temporal_long.py > gpurun_out/ncu_fmha_tlong.log 2>&1
timeout 600 python bench.py --config long --steps 5 --no-cpu-baseline > gpurun_out/bench_long.json 2>&1; cut -c1-200 gpurun_out/bench_long.json
