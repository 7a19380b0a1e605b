"""Developer tool: print the first device/oracle sample mismatches for one case."""
import sys, os
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2405_03488_b200 as A
from oracle_bindings import Oracle

strategy, pattern, gname = sys.argv[1], sys.argv[2], sys.argv[3]
graphs = {"er60_dense": lambda: A.er_graph(60, 0.5, 5).relabel_by_degree(),
          "rmat12_rel": lambda: A.rmat(12, 16, seed=3).relabel_by_degree(),
          "er200": lambda: A.er_graph(200, 0.08, 71)}
g = graphs[gname]()
off, nbr = g.arrays()
A.set_strategy(strategy)
plan = A.compile_plan(pattern)
print(plan.to_dict()["steps"])
v, h, b = A.draw_samples(A.DeviceGraph(g), plan, 9, 12345, 6000)
ov, oh, ob = Oracle().draw_records(off, nbr, g.edge_count, plan, 9, 12345, 6000)
bad = np.nonzero((v != ov) | (b != ob).any(1))[0]
print("mismatches", len(bad))
for i in bad[:8]:
    print(i, "dev", v[i], b[i].tolist(), "orc", ov[i], ob[i].tolist())
    for x in ob[i][:2].tolist() + b[i][:3].tolist():
        if x != 0xffffffff:
            print("   N(%d) =" % x, nbr[off[x]:off[x+1]].tolist())
