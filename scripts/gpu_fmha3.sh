set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x --timeout 100 -k "attention_core_bf16" > gpurun_out/fmha_tests3.log 2>&1; tail -3 gpurun_out/fmha_tests3.log
grep -q "passed" gpurun_out/fmha_tests3.log || exit 1
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_configs.py tests/test_gpu_edge.py -q -x --timeout 300 -k "attention or attn" > gpurun_out/fmha_tests3b.log 2>&1; tail -3 gpurun_out/fmha_tests3b.log
for v in "" pt1 "" pt1; do
  if [ -z "$v" ]; then timeout 120 python scripts/fmha_time.py; else DSP_LIB_OVERRIDE=paper_2403_10266_b200/libdsp_$v.so timeout 120 python scripts/fmha_time.py; fi
done 2>&1 | tee gpurun_out/fmha_ab3.txt
PT=1 DSP_LIB_OVERRIDE=paper_2403_10266_b200/libdsp_trace.so timeout 120 python scripts/fmha_trace.py > gpurun_out/trace_split.txt 2>&1; head -20 gpurun_out/trace_split.txt
timeout 600 python -m pytest tests/test_gpu_transport.py tests/test_gpu_ulysses.py -q --timeout 300 -x > gpurun_out/emul.log 2>&1; tail -3 gpurun_out/emul.log
