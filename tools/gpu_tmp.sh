timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "Error|assert|FAILED|passed|failed" | head -20
QT_SWEEP_DT=f32 QT_SWEEP_BS=16,32 timeout 600 python tools/perf_configs.py leafsweep 2>&1 | tail -14 | cut -c1-200
timeout 300 python tools/perf_configs.py 2 3 5f32 2>&1 | tail -3 | cut -c1-200
