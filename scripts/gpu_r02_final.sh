# Round-2 final evidence: GPU suite, smoke, every bench config, reference arm, launch list, ncu captures,
# per-rank projection, DSP vs Ulysses A/B, switch sweep over virtual ranks
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cut -c1-200 gpurun_out/bench.json
timeout 600 python bench.py --config long --steps 5 > gpurun_out/bench_long.json 2>&1; cut -c1-200 gpurun_out/bench_long.json
timeout 600 python bench.py --config model28 --steps 5 > gpurun_out/bench_model28.json 2>&1; cut -c1-200 gpurun_out/bench_model28.json
timeout 600 python bench.py --config nd --steps 20 > gpurun_out/bench_nd.json 2>&1; cut -c1-200 gpurun_out/bench_nd.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2>&1; cut -c1-200 gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm -s 6 -c 6 -o gpurun_out/prof_block_gemm -f \
   python scripts/block_once.py 2 prep > gpurun_out/ncu_block_gemm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fmha -s 2 -c 2 -o gpurun_out/prof_block_fmha -f \
   python scripts/block_once.py 2 prep > gpurun_out/ncu_block_fmha.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fmha_seq -s 1 -c 1 -o gpurun_out/prof_long_tfmha -f \
   python scripts/block_once_long.py > gpurun_out/ncu_long_tfmha.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm -s 2 -c 1 -o gpurun_out/prof_long_tseq_gemm -f \
   python scripts/block_once_long.py > gpurun_out/ncu_long_tseq_gemm.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:run_copy -c 6 -o gpurun_out/prof_copy -f \
   python scripts/copy_kernels.py > gpurun_out/ncu_copy.log 2>&1
timeout 600 python scripts/project_n.py > gpurun_out/project_n.jsonl 2> gpurun_out/project_n.err; tail -5 gpurun_out/project_n.err
timeout 900 python scripts/ab_schedules.py --prepared > gpurun_out/ab_schedules.jsonl 2>&1; tail -3 gpurun_out/ab_schedules.jsonl
ls -la gpurun_out
