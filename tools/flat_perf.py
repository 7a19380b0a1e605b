"""Developer tool: best-of-N sampling-launch time per 2^24 ids for (strategy, pattern,
graph) combinations, CUDA events on the launching stream, plus a value checksum
so kernel variants can be compared for identical output.

  python tools/flat_perf.py [strategy[,strategy]] [pattern[,pattern]] [graph[,graph]] [reps]
  graphs: rmatNN (relabelled RMAT scale NN, ef16, seed 1), er10k (config 1)
"""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2405_03488_b200 as A  # noqa: E402

strategies = (sys.argv[1] if len(sys.argv) > 1 else "flat").split(",")
patterns = (sys.argv[2] if len(sys.argv) > 2 else "triangle,4clique,5clique").split(",")
graphs = (sys.argv[3] if len(sys.argv) > 3 else "rmat20").split(",")
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
B = 1 << 24
if os.environ.get("AGPM_CORE"):  # dense-core dimension (default 65536)
    A.set_core_dim(int(os.environ["AGPM_CORE"]))
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
vals = torch.empty(B, dtype=torch.float64, device="cuda")
for graph in graphs:
    if graph == "er10k":
        dg = A.DeviceGraph(A.er_graph(10000, 20 / 9999, 1).relabel_by_degree(), stream=st.cuda_stream)
    else:
        dg = A.rmat_device(int(graph[4:]), 16, seed=1, stream=st.cuda_stream)
    dg.prepare()  # dense core + twin-arc index (steady state)
    for strategy in strategies:
        A.set_strategy(strategy)
        for pattern in patterns:
            plan = A.compile_plan(pattern)
            best = 1e9
            for r in range(reps + 1):  # the first launch builds the view indexes
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record(st)
                A.sample_dev(dg, plan, 1, 0, B, vals.data_ptr(), st.cuda_stream)
                e1.record(st)
                torch.cuda.synchronize()
                if r:
                    best = min(best, e0.elapsed_time(e1))
            h = hashlib.sha1(vals.cpu().numpy().tobytes()).hexdigest()[:12]
            print(f"{graph} {strategy:8s} {pattern:8s} {best:8.3f} ms  {B / best * 1e3:.3e} samples/s  "
                  f"hits {(vals != 0).float().mean().item():.4f}  sha {h}", flush=True)
    A.set_strategy("auto")
    del dg
