python tools/perf_configs.py 4 > gpurun_out/p4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_cfg4.csv python tools/perf_configs.py 4 > gpurun_out/ncu_l4.log 2>&1; echo rc=$?
python tools/perf_configs.py 3 > gpurun_out/p3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_cfg3.csv python tools/perf_configs.py 3 > gpurun_out/ncu_l3.log 2>&1; echo rc=$?
