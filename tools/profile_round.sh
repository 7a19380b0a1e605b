#!/bin/bash
# Round profiling recipe (run on the GPU box from the repo root):
#   1. the bench itself (must exit 0 before any ncu run)
#   2. launch list of the bench command (gpu__time_duration, clocks unlocked)
#   3. per-kernel DRAM traffic of 2^24-sample sampling launches (flat sampler)
#   4. one full capture (with source) of the flat sampling kernel (gzipped: the
#      report exceeds gpurun's 64 MiB pull limit uncompressed)
set -e
OUT=gpurun_out/prof
mkdir -p $OUT
python bench.py --steps 10 --warmup 3 > $OUT/bench.log 2>&1
tail -1 $OUT/bench.log > $OUT/bench_line.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_bench.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum \
    --clock-control none --csv --log-file $OUT/sample_dev_traffic.csv python tools/prof_ns.py flat 4clique 2 65536 > $OUT/ncu_traffic.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:fr_flat -s 1 -c 1 -o /tmp/flat_full \
    python tools/prof_ns.py flat 4clique 2 65536 > $OUT/ncu_full.log 2>&1
gzip -c /tmp/flat_full.ncu-rep > $OUT/flat_full.ncu-rep.gz
echo done
