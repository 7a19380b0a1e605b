OUT=gpurun_out/ab
mkdir -p $OUT
python tools/prof_ns.py flat 4clique 2 65536 rmat20 > $OUT/clean.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:fr_flat -s 1 -c 1 -o /tmp/flat_oct -f python tools/prof_ns.py flat 4clique 2 65536 rmat20 > $OUT/ncu.log 2>&1
ncu -i /tmp/flat_oct.ncu-rep --page raw --csv > $OUT/flat_oct2_raw.csv 2>/dev/null
python tools/ncu_raw_summary.py $OUT/flat_oct2_raw.csv oct2 > $OUT/flat_oct2_summary.txt
python tools/ncu_hot.py /tmp/flat_oct.ncu-rep 60 > $OUT/flat_oct2_hot.txt 2>/dev/null
cat $OUT/flat_oct2_summary.txt $OUT/flat_oct2_hot.txt
