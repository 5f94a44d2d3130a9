# full check: GPU tests, bench (all legs), per-config timings
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -2 gpurun_out/bench.log
timeout 600 python tools/perf_configs.py 1 2 3 4 5 dense4096 > gpurun_out/perf_configs.log 2>&1; echo "perf rc=$?"
cat gpurun_out/perf_configs.log
