timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 7000 gpurun_out/bench.log; tail -3 gpurun_out/bench.err
timeout 600 python tools/perf_configs.py 1 3 sym2 sym16 2>&1 | tail -4
