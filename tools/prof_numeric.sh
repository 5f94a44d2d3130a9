# ncu --set full of one numeric-kernel launch per config given in $CFGS
for c in ${CFGS:-4}; do
ncu --set full --clock-control none --import-source on -k regex:k_numeric -s 2 -c 1 -o gpurun_out/prof_${TAG:-x}_$c python tools/perf_configs.py $c > gpurun_out/ncu_${TAG:-x}_$c.log 2>&1; echo "cfg $c rc=$?"
done
