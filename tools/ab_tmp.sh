python -m pytest tests/test_gpu_ns.py -x -q -m gpu -k "sorted_order or twin or prepare" 2>&1 | tail -2
python bench.py --no-cpu-baseline 2>&1 | tail -1 | cut -c1-250
