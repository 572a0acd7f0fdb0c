# ncu --set full captures of the hot kernels at blk N=1 (run under gpurun from the repo root)
set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm -s 4 -c 4 -o gpurun_out/prof_gemm -f \
   python scripts/prof_gemm.py > gpurun_out/ncu_gemm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fmha -s 2 -c 2 -o gpurun_out/prof_fmha -f \
   python scripts/prof_kernels.py fmha > gpurun_out/ncu_fmha.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fmha -s 2 -c 1 -o gpurun_out/prof_fmha_tlong -f \
   python scripts/prof_temporal_long.py > gpurun_out/ncu_fmha_tlong.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:row_stats -s 1 -c 1 -o gpurun_out/prof_rowstats -f \
   python scripts/block_once.py 2 prep > gpurun_out/ncu_rowstats.log 2>&1
ls -la gpurun_out/*.ncu-rep
