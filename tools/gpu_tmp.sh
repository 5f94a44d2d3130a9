timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "Error|assert|FAILED|passed|failed" | head -20
timeout 300 python tools/perf_configs.py 1 2 3 4 5 5f32 2>&1 | tail -6 | cut -c1-230
timeout 900 python bench.py --steps 20 --warmup 5 --no-e2e 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('value',d['value'],'ms',d['ms_per_step'],'num',r['ms_numeric'],'sym',r['ms_symbolic'],'frac',r['frac'],'fp32',d['fp32_variant']['value'],d['fp32_variant']['ms_per_step'])"
