timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "Error|assert|FAILED|passed|failed" | head -20
python tools/async_diag.py 2>&1 | tail -2
timeout 300 python tools/perf_configs.py 1 1async 2 3 2>&1 | tail -4 | cut -c1-200
