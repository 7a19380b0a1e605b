python -m pytest tests/test_gpu_ns.py -x -q -m gpu -k "sorted_order" 2>&1 | tail -2
python tools/flat_perf.py auto triangle,4clique,5clique,6clique,4cycle rmat20 5 2>&1 | grep rmat
python tools/flat_perf.py auto 4clique,5clique rmat18,rmat21 3 2>&1 | grep rmat
python bench.py --no-cpu-baseline 2>&1 | tail -1 | cut -c1-250
