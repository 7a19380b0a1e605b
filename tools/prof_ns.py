"""Developer tool: sample 2^24 ids of the bench workload through one strategy (for ncu)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2405_03488_b200 as A
strategy = sys.argv[1] if len(sys.argv) > 1 else "frontier"
pattern = sys.argv[2] if len(sys.argv) > 2 else "4clique"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
core = int(sys.argv[4]) if len(sys.argv) > 4 else 16384
A.set_core_dim(None if core < 0 else core)  # -1 = auto
graph = sys.argv[5] if len(sys.argv) > 5 else "rmat20"
if graph == "er10k":  # config 1
    g = A.er_graph(10000, 20 / 9999, 1).relabel_by_degree()
    dg = A.DeviceGraph(g)
else:  # built on the device (== the host builder, tests/test_gpu_ingest.py)
    dg = A.rmat_device(int(graph[4:]), 16, seed=1)
plan = A.compile_plan(pattern)
if not os.environ.get("AGPM_NO_PREPARE"):
    dg.prepare()  # steady state: dense core + twin-arc index built before the timed launches
A.set_strategy(strategy)
if os.environ.get("AGPM_RNG"):
    A.set_rng(os.environ["AGPM_RNG"])
B = 1 << 24
vals = torch.empty(B, dtype=torch.float64, device="cuda")
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
for r in range(reps):
    torch.cuda.synchronize(); t = time.perf_counter()
    A.sample_dev(dg, plan, 1, r * B, B, vals.data_ptr(), st.cuda_stream)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"{strategy} core={core} {graph} {pattern} rep {r}: {dt*1e3:.2f} ms  {B/dt:.3e} samples/s  hits {(vals != 0).float().mean().item():.4f}")
