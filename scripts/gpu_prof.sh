set -x
mkdir -p gpurun_out
timeout 300 python scripts/lib_compare.py > gpurun_out/lib_compare.txt 2>&1; cat gpurun_out/lib_compare.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm -s 4 -c 4 -o gpurun_out/prof_gemm -f \
   python scripts/prof_gemm.py > gpurun_out/ncu_gemm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fmha -s 2 -c 2 -o gpurun_out/prof_fmha -f \
   python scripts/prof_kernels.py fmha > gpurun_out/ncu_fmha.log 2>&1
ls -la gpurun_out
