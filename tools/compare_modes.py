"""Eager verify vs lazy verify (NS-base) on the device, config-2 graph.

    python tools/compare_modes.py [pattern ...]

For each pattern: samples/s of one 2^22-sample launch per mode (CUDA events on
a dedicated stream), the hit rate, and run_ns_online(1 %, 5 %) time and n per
mode (lazy capped at 2^28 samples). Prints one JSON line per pattern.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2405_03488_b200 as A  # noqa: E402


def main():
    pats = sys.argv[1:] or ["triangle", "4cycle", "4clique"]
    dg = A.rmat_device(20, 16, seed=1, relabel=True)
    st = torch.cuda.Stream()
    B = 1 << 22
    vals = torch.empty(B, dtype=torch.float64, device="cuda")
    for pat in pats:
        row = {"pattern": pat, "graph": "rmat20_ef16_relabelled"}
        for mode in ("eager", "lazy"):
            plan = A.compile_plan(pat, mode)
            A.sample_dev(dg, plan, 1, 0, B, vals.data_ptr(), st.cuda_stream)  # warm-up
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(st)
            A.sample_dev(dg, plan, 1, B, B, vals.data_ptr(), st.cuda_stream)
            e1.record(st)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            pol = A.OnlinePolicy(max_samples=1 << 28)
            r = A.run_ns_online(dg, plan, 0.01, 0.05, pol, seed=1)
            row[mode] = {"samples_per_s": B / (ms * 1e-3), "hit_rate": (vals != 0).double().mean().item(),
                         "online_seconds": r.seconds, "online_n": r.report.n,
                         "converged": bool(r.report.converged), "estimate": r.report.mu}
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
