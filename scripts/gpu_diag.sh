set -x
mkdir -p gpurun_out
PT=1 DSP_LIB_OVERRIDE=paper_2403_10266_b200/libdsp_trace.so timeout 120 python scripts/fmha_trace.py > gpurun_out/trace_pt.txt 2>&1
DSP_LIB_OVERRIDE=paper_2403_10266_b200/libdsp_tracepair.so timeout 120 python scripts/fmha_trace.py > gpurun_out/trace_pair.txt 2>&1
head -30 gpurun_out/trace_pt.txt; head -20 gpurun_out/trace_pair.txt
timeout 600 python -m pytest tests/test_gpu_transport.py -q --timeout 300 > gpurun_out/pytest_transport.log 2>&1; tail -3 gpurun_out/pytest_transport.log
timeout 600 python scripts/diag_model28.py 13 > gpurun_out/diag28.txt 2>&1; cat gpurun_out/diag28.txt
