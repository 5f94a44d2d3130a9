QT_NUM_PROF=1 timeout 300 python tools/perf_configs.py sym16 2>&1 | grep "numeric prof" | tail -2
QT_NUM_PROF=1 QT_SWEEP_DT=f64 QT_SWEEP_BS=16 timeout 300 python tools/perf_configs.py leafsweep 2>&1 | grep "numeric prof" | tail -3
