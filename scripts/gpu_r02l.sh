# ST-DiT extras (Latte pair, temporal pe, adaLN fold): new tests, then the full suite, bench
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stdit.py -q -x --timeout 400 > gpurun_out/pytest_stdit.log 2>&1; tail -25 gpurun_out/pytest_stdit.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench.json 2> gpurun_out/bench.err; cut -c1-150 gpurun_out/bench.json
