# round-2 evidence refresh after the symbolic-pass and small-read changes:
# bench line, launch lists, BFS kernel captures, per-config timings, leaf
# sweep, small-product and end-to-end device timelines.  The numeric kernels
# are unchanged since tools/gpu_profiles_r2.sh (their captures stay).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python bench.py > gpurun_out/r02_bench.log 2> gpurun_out/r02_bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r02_bench.log
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-cfg2 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-cfg2 > /dev/null 2>&1; echo "ncu-l rc=$?"
for c in 1 3; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r02_launches_cfg$c.csv python tools/perf_configs.py $c > /dev/null 2>&1; echo "ncu-l$c rc=$?"
done
full() {  # name kernel-regex skip perf-args...
  local name=$1 k=$2 s=$3; shift 3
  ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 -o /tmp/$name -f python tools/perf_configs.py "$@" > /dev/null 2>&1
  echo "ncu $name rc=$?"
  python tools/summarize_ncu.py full /tmp/$name.ncu-rep > gpurun_out/$name.json
}
full r02_ncu_full_bfs_large_cfg3 k_bfs_large 2 3
full r02_ncu_full_bfs_large_cfg2 k_bfs_large 2 2
full r02_ncu_full_bfs_small_cfg3 k_bfs_small 2 3
full r02_ncu_full_bfs_small_cfg1 k_bfs_small 2 1
python tools/async_diag.py > gpurun_out/r02_async_cfg1.txt 2>&1
timeout 300 python tools/perf_configs.py 1async 1off >> gpurun_out/r02_async_cfg1.txt 2>&1
timeout 300 python tools/host_cost.py leaf32_0.01 cfg1 >> gpurun_out/r02_async_cfg1.txt 2>&1
timeout 300 python tools/timeline.py leaf32_0.01 cfg1 cfg3 cfg5 2>&1 | grep -v -i warn > gpurun_out/r02_timeline_small.txt
timeout 300 python tools/e2e_timeline.py 6 2>&1 | grep -v -i warn > gpurun_out/r02_timeline_e2e.txt
timeout 1200 python tools/perf_configs.py 1 2 3 4 5 dense4096 5f32 dense4096f32 sym2 sym5f32 sym4 sym16 scr4 virt8 virt8f32 virt4cfg4 virtsym8 virtsym4cfg4 > gpurun_out/r02_perf_configs.jsonl 2>&1; echo "perf rc=$?"
timeout 900 python tools/perf_configs.py leafsweep > gpurun_out/r02_leaf_sweep.jsonl 2>&1; echo "leaf rc=$?"
du -sh gpurun_out
