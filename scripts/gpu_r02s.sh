set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_configs.py tests/test_gpu_edge.py -q -x --timeout 300 -k "attention or attn or cross" > gpurun_out/pytest_fmha.log 2>&1; tail -2 gpurun_out/pytest_fmha.log
for v in "" nodb "" nodb; do
  if [ -z "$v" ]; then timeout 120 python scripts/fmha_time.py; else DSP_LIB_OVERRIDE=paper_2403_10266_b200/libdsp_$v.so timeout 120 python scripts/fmha_time.py; fi
done > gpurun_out/fmha_ab.txt 2>&1; grep spatial gpurun_out/fmha_ab.txt
