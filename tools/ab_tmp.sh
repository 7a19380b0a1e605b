python tools/flat_perf.py flat,frontier 4clique rmat26,rmat27 2 2>&1 | grep rmat
