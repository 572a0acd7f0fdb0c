set -x
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for v in "" ""; do
  timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/b.json 2>/dev/null
  python -c "
import json
d=json.loads([x for x in open('gpurun_out/b.json') if x.startswith('{')][-1]); st=d['stages']
print('$v', d['ms_per_step'], {k: st[k]['us'] for k in ('LN2','QKV_S','QKV_T','PROJ_S','FC1','FC2')})"
done
