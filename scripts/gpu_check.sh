# One gpurun call: the new transport / parity tests first, then the whole GPU suite, smoke, bench.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_transport.py -q --timeout 300 > gpurun_out/pytest_transport.log 2>&1; tail -5 gpurun_out/pytest_transport.log
timeout 1200 python -m pytest tests/test_gpu_configs.py tests/test_gpu_block.py -q --timeout 600 -k "n_invariant or prepared or large_m or model28 or graph" > gpurun_out/pytest_parity.log 2>&1; tail -5 gpurun_out/pytest_parity.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cut -c1-400 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log
