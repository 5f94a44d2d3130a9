# round-2 evidence for profiles/: bench line, launch lists, ncu --set full of the
# numeric kernels (cfg1-5, FP32 cfg5, interior rank of cfg5 P=8), BFS kernels (cfg3, cfg2).
# Reports go to /tmp on the box; only their summaries (and the source pages of two) come back.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python bench.py > gpurun_out/r02_bench.log 2> gpurun_out/r02_bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r02_bench.log
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-cfg2 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-cfg2 > /dev/null 2>&1; echo "ncu-l rc=$?"
for c in 1 3 4; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r02_launches_cfg$c.csv python tools/perf_configs.py $c > /dev/null 2>&1; echo "ncu-l$c rc=$?"
done
full() {  # name kernel-regex skip perf-args...
  local name=$1 k=$2 s=$3; shift 3
  ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 -o /tmp/$name -f python tools/perf_configs.py "$@" > /dev/null 2>&1
  echo "ncu $name rc=$?"
  python tools/summarize_ncu.py full /tmp/$name.ncu-rep > gpurun_out/$name.json
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/$name.raw.csv 2>/dev/null
}
for c in 1 2 3 4 5; do full r02_ncu_full_numeric_cfg$c k_numeric_f64 3 $c; done
full r02_ncu_full_numeric_cfg5_r3of8 k_numeric_f64 3 virt8r3
full r02_ncu_full_numeric_f32_cfg5 k_numeric_f32 2 5f32
full r02_ncu_full_bfs_large_cfg3 k_bfs_large 2 3
full r02_ncu_full_bfs_large_cfg2 k_bfs_large 2 2
full r02_ncu_full_bfs_small_cfg3 k_bfs_small 2 3
for c in 3 4 sym16; do QT_NUM_PROF=1 timeout 300 python tools/perf_configs.py $c 2>&1 | grep "numeric prof" | tail -1; done > gpurun_out/r02_numeric_prof.txt
python tools/async_diag.py > gpurun_out/r02_async_cfg1.txt 2>&1
timeout 300 python tools/perf_configs.py 1async >> gpurun_out/r02_async_cfg1.txt 2>&1
timeout 1200 python tools/perf_configs.py 1 2 3 4 5 dense4096 5f32 dense4096f32 sym2 sym5f32 sym4 sym16 scr4 virt8 virt8f32 virt4cfg4 virtsym8 virtsym4cfg4 > gpurun_out/r02_perf_configs.jsonl 2>&1; echo "perf rc=$?"
timeout 900 python tools/perf_configs.py leafsweep > gpurun_out/r02_leaf_sweep.jsonl 2>&1; echo "leaf rc=$?"
du -sh gpurun_out
