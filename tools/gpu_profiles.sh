# refresh the evidence under profiles/: bench line, launch list, full captures of the
# FP64 and FP32 numeric kernels, per-config timings (all on one B200 via gpurun)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench.log
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/plain_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu1.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_numeric_f64 -s 3 -c 1 -o gpurun_out/prof_numeric_cfg2 -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu2.log 2>&1; echo "ncu2 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_numeric_f32 -s 2 -c 1 -o gpurun_out/prof_numeric_f32_cfg5 -f python tools/perf_configs.py 5f32 > gpurun_out/ncu3.log 2>&1; echo "ncu3 rc=$?"
timeout 1200 python tools/perf_configs.py 1 2 3 4 5 dense4096 5f32 err5f32 dense4096f32 sym2 sym5f32 sym4 sym16 scr4 virt8 virt8f32 virt4cfg4 virtsym8 virtsym4cfg4 > gpurun_out/perf_configs.log 2>&1; echo "perf rc=$?"
timeout 600 python tools/perf_configs.py leafsweep > gpurun_out/leafsweep.log 2>&1; echo "leaf rc=$?"
tail -3 gpurun_out/perf_configs.log
