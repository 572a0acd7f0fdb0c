# TSEQ temporal layout: full GPU suite, A/B timing (block stages), long bench
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 400 > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench.json 2> gpurun_out/bench.err; cut -c1-150 gpurun_out/bench.json
DSP_LIB_OVERRIDE=paper_2403_10266_b200/libdsp_notseq.so timeout 900 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_notseq.json 2>&1; cut -c1-150 gpurun_out/bench_notseq.json
timeout 600 python bench.py --config long --steps 5 --no-cpu-baseline > gpurun_out/bench_long.json 2>&1; cut -c1-150 gpurun_out/bench_long.json
