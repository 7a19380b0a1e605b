"""Developer probe: time to converge (1 %@95 %) per pattern on the config-2 graph."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_03488_b200 as A
dg = A.rmat_device(20, 16, seed=1, relabel=True)
for pat in sys.argv[1:] or ["4clique"]:
    plan = A.compile_plan(pat)
    A.run_ns_online(dg, plan, 0.01, 0.05, A.OnlinePolicy(), seed=1)
    ts = []
    for r in range(5):
        res = A.run_ns_online(dg, plan, 0.01, 0.05, A.OnlinePolicy(), seed=1)
        ts.append(res.seconds)
    print(f"first={os.environ.get('AGPM_ONLINE_FIRST', 65536)} {pat}: n={res.report.n} launched={res.samples_launched} "
          f"best {min(ts)*1e3:.3f} ms median {sorted(ts)[2]*1e3:.3f} ms", flush=True)
