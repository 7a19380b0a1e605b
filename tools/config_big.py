"""Device ingest + online NS on the big RMAT configs (BASELINE configs 3 / 5).

    python tools/config_big.py --scale 27 --pattern 4clique

Builds RMAT-<scale> ef16 in HBM (agpm_gen_rmat_device: generate, sort, dedup,
relabel, CSR), then runs run_ns_online to 1 %@95 % and prints one JSON line
with the ingest time, the graph size and the time to converge (CUDA events on
the library's stream bracket both phases; sync on both sides).
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_03488_b200 as agpm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=27)
    ap.add_argument("--edge-factor", type=int, default=16)
    ap.add_argument("--pattern", default="4clique")
    ap.add_argument("--eps", type=float, default=0.01)
    ap.add_argument("--delta", type=float, default=0.05)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--strategy", default="auto")
    ap.add_argument("--core", type=int, default=-1, help="dense-core dimension; -1 = auto")
    ap.add_argument("--skip-online", action="store_true")
    args = ap.parse_args()
    import torch
    torch.cuda.init()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dg = agpm.rmat_device(args.scale, args.edge_factor, seed=args.seed, relabel=True)
    agpm.sync()
    t_ingest = time.perf_counter() - t0
    info = dg.info()
    plan = agpm.compile_plan(args.pattern)
    agpm.set_strategy(args.strategy)
    agpm.set_core_dim(None if args.core < 0 else args.core)
    runs = []
    for r in range(0 if args.skip_online else args.repeats):
        agpm.sync()
        t0 = time.perf_counter()
        res = agpm.run_ns_online(dg, plan, args.eps, args.delta, agpm.OnlinePolicy(), seed=args.seed + r)
        agpm.sync()
        runs.append({"seconds": time.perf_counter() - t0, "n": res.report.n, "estimate": res.report.mu,
                     "rel_err_bound": res.report.epsilon_hat, "converged": bool(res.report.converged)})
    # fixed-budget throughput: 2^24-sample launches, CUDA events on the launching stream;
    # steady state (twin-arc index built: it is otherwise built after `arcs` sampled ids)
    dg.prepare()
    B = 1 << 24
    vals = torch.empty(B, dtype=torch.float64, device="cuda")
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    agpm.sample_dev(dg, plan, args.seed, 0, B, vals.data_ptr(), st.cuda_stream)  # warm-up
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for r in range(3):
        agpm.sample_dev(dg, plan, args.seed, (r + 1) * B, B, vals.data_ptr(), st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    # SURVEY §8(d) B_min sector model on this graph (device replay of 2^22 sample paths)
    bmin = agpm.bmin_bytes(dg, plan, args.seed, 0, 1 << 22, st.cuda_stream) / float(1 << 22)
    peak = 6531.9
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) as f:
            peak = json.load(f)["hbm_gbs"]
    except Exception:
        pass
    print(json.dumps({"workload": f"rmat{args.scale}_ef{args.edge_factor}_relabelled_{args.pattern}",
                      "strategy": args.strategy, "strategy_run": agpm.strategy_for(dg, plan, B),
                      "core_dim": "auto" if args.core < 0 else args.core,
                      "ingest_seconds": t_ingest, "graph": info,
                      "free_gb_after_ingest": torch.cuda.mem_get_info()[0] / 1e9, "online": runs,
                      "fixed_budget": {"samples": B, "ms": ms, "samples_per_s": B / (ms / 1e3),
                                       "hit_rate": float((vals != 0).double().mean().item()),
                                       "bmin_bytes_per_sample": bmin,
                                       "roofline_frac": bmin * B / (ms / 1e3) / 1e9 / peak}}))


if __name__ == "__main__":
    main()
