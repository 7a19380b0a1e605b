#!/bin/bash
# Round-2 profiling recipe (GPU box, repo root). Every ncu run follows a clean
# run of the same command; numbers printed under ncu are never bench values.
OUT=${OUT:-gpurun_out/prof7}
mkdir -p $OUT
python bench.py --steps 10 --warmup 3 > $OUT/bench.log 2>&1 || exit 1
tail -1 $OUT/bench.log > $OUT/bench_line.json
# 1. launch list of the bench command (cold-cache, serialised per-launch times)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_bench.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum
# 2. per-kernel traffic (auto strategy, auto core): flat 4-clique RMAT-20 (config 2), flat 4-cycle RMAT-22
#    (config 3), frontier 4-clique RMAT-27 (config 5), the 4-cycle pair count (config 3 region split)
python tools/prof_ns.py auto 4clique 2 -1 rmat20 > $OUT/clean_flat.log 2>&1 && \
ncu --metrics $M --clock-control none --csv --log-file $OUT/traffic_flat_rmat20.csv -k 'regex:fr_|flat_seedkey|RadixSort' python tools/prof_ns.py auto 4clique 2 -1 rmat20 > /dev/null 2>&1
python tools/prof_ns.py auto 4cycle 2 -1 rmat22 > $OUT/clean_c3.log 2>&1 && \
ncu --metrics $M --clock-control none --csv --log-file $OUT/traffic_4cycle_rmat22.csv -k regex:fr_ python tools/prof_ns.py auto 4cycle 2 -1 rmat22 > /dev/null 2>&1
python tools/prof_ns.py auto 4clique 2 -1 rmat27 > $OUT/clean_c5.log 2>&1 && \
ncu --metrics $M --clock-control none --csv --log-file $OUT/traffic_4clique_rmat27.csv -k regex:fr_ python tools/prof_ns.py auto 4clique 2 -1 rmat27 > /dev/null 2>&1
python tools/prof_c4.py 22 2 > $OUT/clean_c4.log 2>&1 && \
ncu --metrics $M --clock-control none --csv --log-file $OUT/traffic_c4_rmat22.csv -k regex:c4_ python tools/prof_c4.py 22 1 > /dev/null 2>&1
# 3. full captures (with source): the flat kernel's 2nd launch on config 2 and on config 3, the
#    frontier isect on RMAT-27 4-clique (its 3rd launch = step 1 of the second pass)
ncu --set full --import-source on --clock-control none -k regex:fr_flat -s 1 -c 1 -f -o /tmp/flat_full \
    python tools/prof_ns.py auto 4clique 2 -1 rmat20 > $OUT/ncu_full_flat.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:fr_flat -s 1 -c 1 -f -o /tmp/flat_c3_full \
    python tools/prof_ns.py auto 4cycle 2 -1 rmat22 > $OUT/ncu_full_flat_c3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:fr_isect -s 2 -c 1 -f -o /tmp/isect_full \
    python tools/prof_ns.py auto 4clique 2 -1 rmat27 > $OUT/ncu_full_isect.log 2>&1
for r in flat_full flat_c3_full isect_full; do
  ncu -i /tmp/$r.ncu-rep --page raw --csv > $OUT/${r}_raw.csv 2>/dev/null
  python tools/ncu_hot.py /tmp/$r.ncu-rep 40 > $OUT/${r}_hot.txt 2>/dev/null
done
echo done
