for m in 8192 4096 2048 1024; do echo "maxF $m"; export QT_SMALL_MAXF=$m; python tools/bs16_small.py 0.01 16 2>&1 | tail -1; python tools/bs16_small.py 0.05 16 2>&1 | tail -1; python tools/bs16_small.py 0.02 32 2>&1 | tail -1; timeout 300 python tools/perf_configs.py 1 2 3 4 2>&1 | tail -4 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['config'][:20], d['ms_step'], d['ms_symbolic'])"; done
