# round-2 profiling: host-side phase trace (cfg1, cfg3), launch lists, full captures of the
# BFS kernels and cfg3's numeric kernel, numeric traffic for cfg5 P=1 and an interior rank
set -x
QT_TRACE=1 timeout 300 python tools/perf_configs.py 1 3 > gpurun_out/trace_perf.log 2> gpurun_out/trace.err; echo "trace rc=$?"
grep -v "^\[qt trace\]" gpurun_out/trace.err | tail -3
tail -3 gpurun_out/trace.err
cat gpurun_out/trace_perf.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg1.csv python tools/perf_configs.py 1 > /dev/null 2>&1; echo "ncu-l1 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg3.csv python tools/perf_configs.py 3 > /dev/null 2>&1; echo "ncu-l3 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_bfs_large -s 2 -c 1 -o gpurun_out/prof_bfs_large_cfg3 -f python tools/perf_configs.py 3 > gpurun_out/ncu_b1.log 2>&1; echo "ncu-bl rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_bfs_small -s 2 -c 1 -o gpurun_out/prof_bfs_small_cfg3 -f python tools/perf_configs.py 3 > gpurun_out/ncu_b2.log 2>&1; echo "ncu-bs rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_numeric_f64 -s 3 -c 1 -o gpurun_out/prof_numeric_cfg3 -f python tools/perf_configs.py 3 > gpurun_out/ncu_n3.log 2>&1; echo "ncu-n3 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_numeric_f64 -s 3 -c 1 -o gpurun_out/prof_numeric_cfg5 -f python tools/perf_configs.py 5 > gpurun_out/ncu_n5.log 2>&1; echo "ncu-n5 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_numeric_f64 -s 3 -c 1 -o gpurun_out/prof_numeric_cfg5_r3of8 -f python tools/perf_configs.py virt8r3 > gpurun_out/ncu_n58.log 2>&1; echo "ncu-n58 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_numeric_f64 -s 3 -c 1 -o gpurun_out/prof_numeric_cfg1 -f python tools/perf_configs.py 1 > gpurun_out/ncu_n1.log 2>&1; echo "ncu-n1 rc=$?"
