for c in 262144 524288; do echo "== core $c"; AGPM_CORE=$c python tools/flat_perf.py flat 4cycle,4clique rmat23,rmat24,rmat25 3 2>&1 | grep -E "rmat|rror"; done
