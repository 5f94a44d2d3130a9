# ncu --set full of one launch of kernel regex $K (skip $S launches) under perf_configs $CFG
ncu --set full --clock-control none --import-source on -k regex:${K} -s ${S:-2} -c 1 -o gpurun_out/prof_${TAG:-k}_${CFG} python tools/perf_configs.py ${CFG} > gpurun_out/ncu_${TAG:-k}_${CFG}.log 2>&1; echo "rc=$?"
