"""Developer probe: per-phase timing of the bench's e2e loop (upload / run / free)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_03488_b200 as A
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); sptr = stream.cuda_stream
g = A.rmat(20, 16, seed=1).relabel_by_degree()
plan = A.compile_plan("4clique")
dg = A.DeviceGraph(g, stream=sptr)
B = 1 << 24
values = torch.empty(B, dtype=torch.float64, device="cuda")
if "--prelude" in sys.argv:
    A.bmin_bytes(dg, plan, 1, 0, 1 << 22, sptr)
    for s in range(5):
        A.sample_dev(dg, plan, 1, s * B, B, values.data_ptr(), sptr)
    torch.cuda.synchronize()
g.pin()
A.run_fixed_budget(A.DeviceGraph(g), plan, 1 << 16, 1)
torch.cuda.synchronize()
for s in range(4):
    t1 = time.perf_counter(); d2 = A.DeviceGraph(g); t2 = time.perf_counter()
    A.run_fixed_budget(d2, plan, B, 1 + s); t3 = time.perf_counter()
    del d2; t4 = time.perf_counter()
    print(f"step {s}: upload {(t2-t1)*1e3:.2f} ms  run {(t3-t2)*1e3:.2f} ms  free {(t4-t3)*1e3:.2f} ms", flush=True)
