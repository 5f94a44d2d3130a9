timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "Error|assert|FAILED|passed|failed" | head -20
timeout 300 python tools/perf_configs.py 1 2 3 4 2>&1 | tail -4 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['config'][:20], d['ms_step'], d['ms_symbolic'], d['ms_numeric'])"
QT_BFS_PROF=1 timeout 100 python tools/perf_configs.py 3 2>&1 | grep -A7 "bfs_large" | tail -7
