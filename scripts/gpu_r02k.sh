# seq kernel for block-diagonal tiles (T=16): attention tests, A/B timing, full suite, bench
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_edge.py -q -x --timeout 400 -k "attention or attn or ragged" > gpurun_out/pytest_fmha.log 2>&1; tail -3 gpurun_out/pytest_fmha.log
for v in "" nodiag "" nodiag; do
  if [ -z "$v" ]; then timeout 120 python scripts/fmha_time.py; else DSP_LIB_OVERRIDE=paper_2403_10266_b200/libdsp_$v.so timeout 120 python scripts/fmha_time.py; fi
done > gpurun_out/fmha_ab.txt 2>&1; grep spatial gpurun_out/fmha_ab.txt
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 400 > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench.json 2> gpurun_out/bench.err; cut -c1-150 gpurun_out/bench.json
