# round-2 evidence for profiles/: bench line, launch lists, ncu --set full of the
# numeric kernels (cfg1-5, FP32 cfg5, interior rank of cfg5 P=8), BFS kernels (cfg3, cfg2)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python bench.py > gpurun_out/r02_bench.log 2> gpurun_out/r02_bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r02_bench.log
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-cfg2 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-cfg2 > /dev/null 2>&1; echo "ncu-l rc=$?"
for c in 1 3 4; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r02_launches_cfg$c.csv python tools/perf_configs.py $c > /dev/null 2>&1; echo "ncu-l$c rc=$?"
done
for c in 1 2 3 4 5; do
  ncu --set full --clock-control none --import-source on -k regex:k_numeric_f64 -s 3 -c 1 -o gpurun_out/r02_prof_numeric_cfg$c -f python tools/perf_configs.py $c > /dev/null 2>&1; echo "ncu-n$c rc=$?"
done
ncu --set full --clock-control none --import-source on -k regex:k_numeric_f64 -s 3 -c 1 -o gpurun_out/r02_prof_numeric_cfg5_r3of8 -f python tools/perf_configs.py virt8r3 > /dev/null 2>&1; echo "ncu-n58 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_numeric_f32 -s 2 -c 1 -o gpurun_out/r02_prof_numeric_f32_cfg5 -f python tools/perf_configs.py 5f32 > /dev/null 2>&1; echo "ncu-f32 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_bfs_large -s 2 -c 1 -o gpurun_out/r02_prof_bfs_large_cfg3 -f python tools/perf_configs.py 3 > /dev/null 2>&1; echo "ncu-bl3 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_bfs_large -s 2 -c 1 -o gpurun_out/r02_prof_bfs_large_cfg2 -f python tools/perf_configs.py 2 > /dev/null 2>&1; echo "ncu-bl2 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_bfs_small -s 2 -c 1 -o gpurun_out/r02_prof_bfs_small_cfg3 -f python tools/perf_configs.py 3 > /dev/null 2>&1; echo "ncu-bs3 rc=$?"
for c in 3 4; do QT_NUM_PROF=1 timeout 300 python tools/perf_configs.py $c 2>&1 | grep "numeric prof" | tail -1; done > gpurun_out/r02_numeric_prof.txt
timeout 1200 python tools/perf_configs.py 1 2 3 4 5 dense4096 5f32 dense4096f32 sym2 sym5f32 sym4 sym16 scr4 virt8 virt8f32 virt4cfg4 virtsym8 virtsym4cfg4 > gpurun_out/r02_perf_configs.jsonl 2>&1; echo "perf rc=$?"
timeout 900 python tools/perf_configs.py leafsweep > gpurun_out/r02_leaf_sweep.jsonl 2>&1; echo "leaf rc=$?"
