timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "Error|assert|FAILED|passed|failed" | head -30
QT_SWEEP_DT=f64 QT_SWEEP_BS=16,32 timeout 600 python tools/perf_configs.py leafsweep 2>&1 | tail -14 | cut -c1-200
