python -m pytest tests/test_gpu_ns.py tests/test_gpu_configs.py tests/test_gpu_multi.py tests/test_gpu_scale.py -x -q -m gpu 2>&1 | tail -3
python bench.py 2>&1 | tail -1 > gpurun_out/bench_dedup.json; cut -c1-250 gpurun_out/bench_dedup.json
