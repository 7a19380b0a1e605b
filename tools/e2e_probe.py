"""Developer probe: per-phase timing of the bench's e2e loop (upload / run / free)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_03488_b200 as A
if os.environ.get("E2E_NOGC"):
    import gc
    gc.disable()
if os.environ.get("E2E_CORE"):
    A.set_core_dim(int(os.environ["E2E_CORE"]))
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
import subprocess
smi = None
if "--smi" in sys.argv:  # the bench's clock sampler running alongside
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", "100"],
                           stdout=subprocess.DEVNULL)
    time.sleep(0.5)
for s in range(int(os.environ.get("E2E_STEPS", "4"))):
    t1 = time.perf_counter(); d2 = A.DeviceGraph(g); t2 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); A.run_fixed_budget(d2, plan, B, 1 + s); e1.record(); t3 = time.perf_counter()
    torch.cuda.synchronize(); gpu_ms = e0.elapsed_time(e1)
    del d2; t4 = time.perf_counter()
    print(f"step {s}: upload {(t2-t1)*1e3:.2f} ms  run {(t3-t2)*1e3:.2f} ms  free {(t4-t3)*1e3:.2f} ms  events {gpu_ms:.2f} ms", flush=True)
if smi:
    smi.terminate()
