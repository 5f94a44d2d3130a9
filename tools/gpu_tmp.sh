timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | grep -E "passed|failed"
timeout 300 python tools/perf_configs.py 1 2 3 4 2>&1 | tail -4 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['config'][:20], d['ms_step'], d['ms_symbolic'], d['ms_numeric'])"
QT_NUM_PROF=1 timeout 300 python tools/perf_configs.py 3 2>&1 | grep "numeric prof" | tail -1
