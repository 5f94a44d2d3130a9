QT_BFS_PROF=1 timeout 100 python tools/perf_configs.py 1 2>&1 | grep bfs_small | tail -1
timeout 300 python tools/perf_configs.py 1 3 2>&1 | tail -2
