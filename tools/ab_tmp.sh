python -m pytest tests/test_gpu_scale.py tests/test_gpu_ns.py tests/test_gpu_configs.py tests/test_gpu_multi.py -x -q -m gpu 2>&1 | tail -3
python tools/flat_perf.py auto 4clique,5clique rmat20,rmat22,rmat24 3 2>&1 | grep rmat
