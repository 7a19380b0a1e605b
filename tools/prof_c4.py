"""Developer tool: the config-3 region split (RMAT-22 ef16 relabelled, 4-cycle,
tau = 64) with the exact dense leg, for ncu captures of the cycle4_sparse kernels."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2405_03488_b200 as A  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
dg = A.rmat_device(scale, 16, seed=1)
plan = A.compile_plan("4cycle")
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    r = A.region_split(dg, plan, 64, dense="ns")
    print(f"rmat{scale} c_sparse {r.c_sparse} sparse {r.sparse_seconds:.3f} s")
