mkdir -p gpurun_out
export CUDA_MODULE_LOADING=EAGER
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_memcheck_smoke.log 2>&1; echo rc=$? >> gpurun_out/san_memcheck_smoke.log
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 20 python -m pytest -q -x tests/test_gpu_kernels.py -k "linear or (attention_core_bf16 and (16-64 or 5-16 or 2-70))" > gpurun_out/san_memcheck_kernels.log 2>&1; echo rc=$? >> gpurun_out/san_memcheck_kernels.log
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool synccheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_synccheck_smoke.log 2>&1; echo rc=$? >> gpurun_out/san_synccheck_smoke.log
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_racecheck_smoke.log 2>&1; echo rc=$? >> gpurun_out/san_racecheck_smoke.log
