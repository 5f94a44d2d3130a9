# quick GPU iteration: parity subset + bench without the slow legs
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "random_patterns or cfg1 or cfg2 or virtual or identity" 2>&1 | tail -3
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('value',d['value'],'ms',d['ms_per_step'],'num',r['ms_numeric'],'sym',r['ms_symbolic'],'frac',r['frac'],'peak',r['peak'],'clk',d['clocks'])"
