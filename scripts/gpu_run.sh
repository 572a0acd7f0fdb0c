timeout 900 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -3
for pdl in 1 0; do DSP_PDL=$pdl timeout 300 python bench.py --steps 30 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('PDL=$pdl', d['ms_per_step'], d['block_roofline']['frac'])"; done
timeout 300 python scripts/project_n.py | cut -c1-200
