# spatial FMHA A/B: P in TMEM (fmha_pt_kernel, default) vs the shared-memory-P pair kernel
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_configs.py tests/test_gpu_edge.py -q -x --timeout 300 -k "attention or attn" > gpurun_out/fmha_tests.log 2>&1; tail -3 gpurun_out/fmha_tests.log
for v in "" pairsmem "" pairsmem; do
  if [ -z "$v" ]; then timeout 120 python scripts/fmha_time.py; else DSP_LIB_OVERRIDE=paper_2403_10266_b200/libdsp_$v.so timeout 120 python scripts/fmha_time.py; fi
done 2>&1 | tee gpurun_out/fmha_ab2.txt
timeout 600 python -m pytest tests/test_gpu_block.py tests/test_gpu_configs.py -q --timeout 300 -k "model28 or blk_prepared or block_bf16" > gpurun_out/block_tests.log 2>&1; tail -3 gpurun_out/block_tests.log
timeout 900 python bench.py > gpurun_out/bench2.json 2> gpurun_out/bench2.err; tail -3 gpurun_out/bench2.err
python -c "
import json; d=json.loads(open('gpurun_out/bench2.json').read().strip().splitlines()[-1])
print('block', d['ms_per_step'], d['block_roofline']); print('roof', d['roofline'])
for k,v in d['stages'].items(): print(k, v.get('us'), v.get('event_us'), v.get('frac'))
"
