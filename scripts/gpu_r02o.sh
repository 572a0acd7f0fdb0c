set -x
for v in "" prevuv "" prevuv; do
  if [ -z "$v" ]; then timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/b.json 2>/dev/null; else DSP_LIB_OVERRIDE=paper_2403_10266_b200/libdsp_$v.so timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/b.json 2>/dev/null; fi
  python -c "
import json
d=json.loads([x for x in open('gpurun_out/b.json') if x.startswith('{')][-1]); st=d['stages']
print('$v', d['ms_per_step'], {k: st[k]['us'] for k in ('QKV_S','QKV_T','PROJ_S','FC1','FC2')})"
done
