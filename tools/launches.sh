# ncu launch list (per-kernel device time) for perf_configs ${CFG}
ncu --metrics gpu__time_duration.sum --clock-control none -c ${COUNT:-400} --csv --log-file gpurun_out/launches_${CFG}.csv python tools/perf_configs.py ${CFG} > gpurun_out/ncu_l_${CFG}.log 2>&1; echo "rc=$?"
