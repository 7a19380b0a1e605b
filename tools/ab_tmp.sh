for v in _old ""; do echo "== variant '$v'"; AGPM_LIB=$PWD/paper_2405_03488_b200/libagpm_b200$v.so python tools/flat_perf.py flat triangle,4clique,5clique,4cycle rmat20 5 2>&1 | grep rmat; done
python tools/flat_perf.py auto 4cycle,4clique rmat22 3 2>&1 | grep rmat
