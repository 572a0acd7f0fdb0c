set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k attention 2>&1 | tail -3
for v in "" nopp nosplit p8 "" nopp; do
  if [ -z "$v" ]; then timeout 120 python scripts/fmha_time.py; else DSP_LIB_OVERRIDE=paper_2403_10266_b200/libdsp_$v.so timeout 120 python scripts/fmha_time.py; fi
done 2>&1 | tee gpurun_out/fmha_ab.txt
DSP_LIB_OVERRIDE=paper_2403_10266_b200/libdsp_trace.so timeout 120 python scripts/fmha_trace.py > gpurun_out/fmha_trace.txt 2>&1
