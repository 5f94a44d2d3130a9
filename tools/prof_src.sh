# ncu --set full of one launch of kernel regex $K (skip $S) under `tools/timeline.py $W`;
# brings back the raw page and the per-source-line (CUDA + SASS) stall tables
R=/tmp/prof_${TAG:-k}
ncu -f --set full --warp-sampling-interval ${WSI:-auto} --clock-control none --import-source on -k regex:${K} -s ${S:-2} -c 1 -o $R python tools/timeline.py ${W} > gpurun_out/ncu_${TAG:-k}.log 2>&1; echo "ncu rc=$?"
ncu -i $R.ncu-rep --page raw --csv > gpurun_out/raw_${TAG:-k}.csv 2>&1
ncu -i $R.ncu-rep --page source --csv --print-source cuda > gpurun_out/src_${TAG:-k}.csv 2>&1
ncu -i $R.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_${TAG:-k}.csv 2>&1
ls -la gpurun_out/*${TAG:-k}*
[ -n "$KEEP" ] && cp $R.ncu-rep gpurun_out/ && ls -la gpurun_out/*.ncu-rep
