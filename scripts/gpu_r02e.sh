# FMHA pt variants (exp split), GEMM timing, GPU suite, bench
set -x
mkdir -p gpurun_out
for v in "" p4 p8 sp6 sp8 ""; do
  if [ -z "$v" ]; then timeout 120 python scripts/fmha_time.py; else DSP_LIB_OVERRIDE=paper_2403_10266_b200/libdsp_$v.so timeout 120 python scripts/fmha_time.py; fi
done > gpurun_out/fmha_ab.txt 2>&1; grep spatial gpurun_out/fmha_ab.txt
timeout 300 python scripts/gemm_graph_time.py > gpurun_out/gemm_time.txt 2>&1; cat gpurun_out/gemm_time.txt
timeout 900 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench.json 2> gpurun_out/bench.err; cut -c1-200 gpurun_out/bench.json
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 400 > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log
