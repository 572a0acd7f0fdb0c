# DSP vs Ulysses on the same kernels (virtual ranks), per-rank projection, GEMM shapes
set -x
mkdir -p gpurun_out
timeout 300 python scripts/gemm_graph_time.py > gpurun_out/gemm_time.txt 2>&1; cat gpurun_out/gemm_time.txt
timeout 900 python scripts/ab_schedules.py --prepared > gpurun_out/ab_schedules.jsonl 2>&1; cat gpurun_out/ab_schedules.jsonl
timeout 600 python scripts/project_n.py > gpurun_out/project_n.jsonl 2> gpurun_out/project_n.err; tail -6 gpurun_out/project_n.err
