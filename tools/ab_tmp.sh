mkdir -p gpurun_out/r2e
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2e/smoke.log 2>&1; tail -2 gpurun_out/r2e/smoke.log
python -m pytest tests -x -q -m gpu > gpurun_out/r2e/gputest.log 2>&1; tail -3 gpurun_out/r2e/gputest.log
python bench.py > gpurun_out/r2e/bench.log 2>&1; tail -1 gpurun_out/r2e/bench.log | cut -c1-300
python tools/config_big.py --scale 27 --pattern 4clique > gpurun_out/r2e/config_big27.jsonl 2> gpurun_out/r2e/config_big27.err
grep -o '"online.*' gpurun_out/r2e/config_big27.jsonl | cut -c1-700
