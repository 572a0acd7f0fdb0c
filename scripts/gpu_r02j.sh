# TSEQ (T >= 64 only): new tests, full suite, blk + long bench
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_block.py -q -x --timeout 400 -k tseq > gpurun_out/pytest_tseq.log 2>&1; tail -3 gpurun_out/pytest_tseq.log
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 400 > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench.json 2> gpurun_out/bench.err; cut -c1-150 gpurun_out/bench.json
timeout 600 python bench.py --config long --steps 5 --no-cpu-baseline > gpurun_out/bench_long.json 2>&1; cut -c1-150 gpurun_out/bench_long.json
DSP_LIB_OVERRIDE=paper_2403_10266_b200/libdsp_notseq.so timeout 600 python bench.py --config long --steps 5 --no-cpu-baseline > gpurun_out/bench_long_notseq.json 2>&1; cut -c1-150 gpurun_out/bench_long_notseq.json
