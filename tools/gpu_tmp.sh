timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "Error|assert|FAILED|passed|failed" | head -20
QT_SWEEP_DT=f64 QT_SWEEP_BS=16 timeout 600 python tools/perf_configs.py leafsweep sym16 2>&1 | tail -8 | cut -c1-220
timeout 300 python tools/perf_configs.py 2 3 2>&1 | tail -2 | cut -c1-200
