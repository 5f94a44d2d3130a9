# iteration: GPU parity tests + per-config timings
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/gpu_tests.log
timeout 600 python tools/perf_configs.py ${PERF_CFGS:-1 2 3 4 5 dense4096} > gpurun_out/perf_configs.log 2>&1; echo "perf rc=$?"
cat gpurun_out/perf_configs.log
