mkdir -p gpurun_out/r2d
for v in "" _l1 _l2; do echo "== variant '$v'"; AGPM_LIB=$PWD/paper_2405_03488_b200/libagpm_b200$v.so python tools/flat_perf.py flat triangle,4clique,5clique,4cycle rmat20 5 2>&1 | grep rmat; done
python tools/config_big.py --scale 27 --pattern 4clique > gpurun_out/r2d/config_big27.jsonl 2> gpurun_out/r2d/config_big27.err
python tools/config_big.py --scale 27 --pattern 4cycle >> gpurun_out/r2d/config_big27.jsonl 2>> gpurun_out/r2d/config_big27.err
grep -o '"fixed_budget.*' gpurun_out/r2d/config_big27.jsonl; grep -o '"online.*"fixed' gpurun_out/r2d/config_big27.jsonl | cut -c1-300; tail -3 gpurun_out/r2d/config_big27.err
