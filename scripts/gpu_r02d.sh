# A/B: GEMM epilogue warpgroups / tail split / FC1 BN; FMHA variants + clock64 traces
set -x
mkdir -p gpurun_out
for v in "" wg1 nosplit bn192fc1; do
  if [ -z "$v" ]; then timeout 300 python scripts/gemm_graph_time.py; else DSP_LIB_OVERRIDE=paper_2403_10266_b200/libdsp_$v.so timeout 300 python scripts/gemm_graph_time.py; fi
done > gpurun_out/gemm_ab.txt 2>&1; cat gpurun_out/gemm_ab.txt
for v in "" pt1 pair; do
  if [ -z "$v" ]; then timeout 120 python scripts/fmha_time.py; else DSP_LIB_OVERRIDE=paper_2403_10266_b200/libdsp_$v.so timeout 120 python scripts/fmha_time.py; fi
done > gpurun_out/fmha_ab.txt 2>&1; cat gpurun_out/fmha_ab.txt
PT=1 DSP_LIB_OVERRIDE=paper_2403_10266_b200/libdsp_tracept.so timeout 120 python scripts/fmha_trace.py > gpurun_out/trace_pt.txt 2>&1; head -45 gpurun_out/trace_pt.txt
PT=1 DSP_LIB_OVERRIDE=paper_2403_10266_b200/libdsp_trace.so timeout 120 python scripts/fmha_trace.py > gpurun_out/trace_split.txt 2>&1; head -45 gpurun_out/trace_split.txt
timeout 900 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench.json 2> gpurun_out/bench.err; cut -c1-200 gpurun_out/bench.json
