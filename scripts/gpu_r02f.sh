# GPU suite, bench (blk default with cpu baseline), GEMM timing, ncu launch list + full captures for profiles/r02
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 400 > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cut -c1-200 gpurun_out/bench.json
timeout 300 python scripts/gemm_graph_time.py > gpurun_out/gemm_time.txt 2>&1; cat gpurun_out/gemm_time.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm -s 6 -c 6 -o gpurun_out/prof_block_gemm -f \
   python scripts/block_once.py 2 prep > gpurun_out/ncu_block_gemm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fmha -s 2 -c 2 -o gpurun_out/prof_block_fmha -f \
   python scripts/block_once.py 2 prep > gpurun_out/ncu_block_fmha.log 2>&1
timeout 600 python bench.py --config long --steps 5 --no-cpu-baseline > gpurun_out/bench_long.json 2>&1; cut -c1-200 gpurun_out/bench_long.json
