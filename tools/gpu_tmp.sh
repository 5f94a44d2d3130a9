QT_FUZZ_MUL=600 QT_FUZZ_MISC=150 QT_FUZZ_NBR=100 timeout 2400 python -m pytest tests/test_gpu_fuzz.py -x -q 2>&1 | grep -E "Error|assert|FAILED|passed|failed" | head -20
