python -m pytest tests/test_gpu_ns.py tests/test_gpu_configs.py tests/test_gpu_multi.py -x -q -m gpu 2>&1 | tail -4
python bench.py --no-cpu-baseline 2>&1 | tail -1 | cut -c1-250
python tools/flat_perf.py auto triangle,4clique,5clique,6clique,4cycle rmat20,rmat21 5 2>&1 | grep rmat
