timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "Error|assert|FAILED|passed|failed" | head -30
for c in 3 4; do QT_NUM_PROF=1 timeout 300 python tools/perf_configs.py $c 2>&1 | grep "numeric prof" | tail -1; done
