"""BASELINE.json config 3 end to end: 4-cycle on RMAT-22 ef16 (relabelled).

    python tools/config3.py [--scale 22] [--check-scale 20] [--tau 64]

One JSON line per stage, each timed on the device (the calls synchronise):
  * ns_online      eager-verify NS to 1 %@95 % (the fine-grained scheme);
  * hybrid         the reference's loose-mode selector (fast_profile on a 10 %
                   Bernoulli graph, gamma probing, keep probability, cost cone vs
                   GS model) and the scheme it picks;
  * region_split   builder-defined dense/sparse split: exact
                   count of the 4-cycles touching {deg < tau}, NS on the dense
                   region;
  * accuracy       at --check-scale (default RMAT-20): the device exact count
                   beside the NS and region-split estimates — the relative
                   error must sit inside the 1 % bound.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_03488_b200 as A  # noqa: E402


def timed(fn):
    A.sync()
    t = time.perf_counter()
    out = fn()
    A.sync()
    return time.perf_counter() - t, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=22)
    ap.add_argument("--check-scale", type=int, default=20)
    ap.add_argument("--tau", type=int, default=64)
    ap.add_argument("--pattern", default="4cycle")
    args = ap.parse_args()
    plan = A.compile_plan(args.pattern)
    for scale, check in ((args.check_scale, True), (args.scale, False)):
        t_gen, g = timed(lambda: A.rmat(scale, 16, seed=1).relabel_by_degree())
        dg = A.DeviceGraph(g)
        wl = f"rmat{scale}_ef16_relabelled_{args.pattern}"
        dg.prepare()  # steady state: dense core and twin-arc index built
        for w in range(2):  # warm-up
            A.run_ns_online(dg, plan, 0.01, 0.05, A.OnlinePolicy(), seed=2 + w)
        t_ns, ns = timed(lambda: A.run_ns_online(dg, plan, 0.01, 0.05, A.OnlinePolicy(), seed=1))
        print(json.dumps({"workload": wl, "stage": "ns_online", "seconds": t_ns, "estimate": ns.report.mu,
                          "n": ns.report.n, "epsilon_hat": ns.report.epsilon_hat,
                          "converged": bool(ns.report.converged)}), flush=True)
        t_hy, hy = timed(lambda: A.count_hybrid(g, dg, plan, 0.01, 0.95, seed=1))
        print(json.dumps({"workload": wl, "stage": "hybrid", "seconds": t_hy,
                          "decision": "GS" if hy.decision else "NS", "estimate": hy.estimate,
                          "gamma": hy.gamma, "keep_probability": hy.keep.p,
                          "ns_cone_lower_s": hy.cone.lower_time, "gs_model_s": hy.gs_model.total_seconds}),
              flush=True)
        t_rs, rs = timed(lambda: A.region_split(dg, plan, args.tau, dense="ns", eps=0.01, delta=0.05, seed=1))
        print(json.dumps({"workload": wl, "stage": "region_split", "tau_degree": args.tau, "seconds": t_rs,
                          "sparse_seconds": rs.sparse_seconds, "dense_seconds": rs.dense_seconds,
                          "sparse_vertices": rs.sparse_vertices, "dense_vertices": rs.dense_vertices,
                          "c_sparse": rs.c_sparse, "c_dense": rs.c_dense, "estimate": rs.estimate,
                          "dense_epsilon_hat": rs.dense_epsilon_hat}), flush=True)
        if check:
            t_ex, exact = timed(lambda: A.exact_count(dg, plan))
            print(json.dumps({"workload": wl, "stage": "accuracy", "exact": exact, "exact_seconds": t_ex,
                              "ns_rel_err": abs(ns.report.mu - exact) / exact,
                              "hybrid_rel_err": abs(hy.estimate - exact) / exact,
                              "region_rel_err": abs(rs.estimate - exact) / exact,
                              "bound": 0.01}), flush=True)
        del dg


if __name__ == "__main__":
    main()
