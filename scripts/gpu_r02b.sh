# Round-2 call b: Ulysses N=8 tests, per-rank projection, ncu --set full of the block's GEMMs and FMHAs (prepared path).
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ulysses.py -q --timeout 300 > gpurun_out/pytest_ulysses.log 2>&1; tail -3 gpurun_out/pytest_ulysses.log
timeout 600 python scripts/project_n.py > gpurun_out/project_n.jsonl 2> gpurun_out/project_n.err; tail -6 gpurun_out/project_n.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm -s 6 -c 6 -o gpurun_out/prof_block_gemm -f \
   python scripts/block_once.py 2 prep > gpurun_out/ncu_block_gemm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fmha -s 2 -c 2 -o gpurun_out/prof_block_fmha -f \
   python scripts/block_once.py 2 prep > gpurun_out/ncu_block_fmha.log 2>&1
ls -la gpurun_out/*.ncu-rep
