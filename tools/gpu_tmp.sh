timeout 900 python -m pytest tests/test_gpu_bs16.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -3
QT_SWEEP_DT=f64 QT_SWEEP_BS=16,32 timeout 600 python tools/perf_configs.py leafsweep sym16 2>&1 | tail -16
