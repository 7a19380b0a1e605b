#!/bin/bash
# Round profiling recipe (run on the GPU box from the repo root):
#   1. the bench itself (must exit 0 before any ncu run)
#   2. launch list of the bench command (gpu__time_duration, clocks unlocked)
#   3. per-kernel DRAM traffic of one 2^24-sample sampling launch
#   4. one full capture (with source) of each frontier kernel of one sub-batch
set -e
OUT=gpurun_out/prof
mkdir -p $OUT
python bench.py --steps 10 --warmup 3 > $OUT/bench.log 2>&1
tail -1 $OUT/bench.log > $OUT/bench_line.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_bench.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $OUT/sample_dev_traffic.csv python tools/prof_ns.py frontier 4clique 2 > $OUT/ncu_traffic.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:fr_ -c 5 -o $OUT/frontier_full \
    python tools/prof_ns.py frontier 4clique 1 > $OUT/ncu_full.log 2>&1
echo done
