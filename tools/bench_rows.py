"""Secondary measurements: every §8 row with a device kernel, timed on the device
and beside the compiled reference on the host cores, results compared.

    python tools/bench_rows.py [--quick] [--full]

One JSON line per row: device seconds (best of 3 after a warm-up, the call
synchronises), reference seconds (one run, threads = host cores), equal: bool.
The reference runs through oracle/_ref (the unmodified reference library), so
this needs the built oracle/_ref/libagpm_ref.so (it travels with the repo).
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2405_03488_b200 as A  # noqa: E402
from oracle_bindings import RefLib  # noqa: E402


def best(fn, reps=3):
    fn()
    ts = []
    out = None
    for _ in range(reps):
        t = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - t)
    return min(ts), out


def once(fn):
    t = time.perf_counter()
    out = fn()
    return time.perf_counter() - t, out


def emit(row, **kw):
    print(json.dumps({"row": row, **kw}), flush=True)


def main():
    quick = "--quick" in sys.argv
    threads = os.cpu_count() or 1
    R = RefLib()
    scale = 16 if quick else 18

    # graph for the counting rows: RMAT-<scale> ef16, degree-relabelled
    g = A.rmat(scale, 16, seed=1).relabel_by_degree()
    off, nbr = g.arrays()
    rg = R.from_csr(off, nbr, g.edge_count)
    dg = A.DeviceGraph(g)
    gname = f"rmat{scale}_ef16_relabelled"

    # row 14: exact_count (exact_engine.cpp:66-91), 4-clique and 4-cycle
    for pat in ("4clique", "4cycle"):
        plan = A.compile_plan(pat)
        td, dev = best(lambda: A.exact_count(dg, plan))
        row = dict(graph=gname, pattern=pat, device_s=td, count=dev)
        if pat == "4clique" or "--full" in sys.argv:  # the 4-cycle reference run takes ~11 min on 16 cores
            tr, ref = once(lambda: R.exact_count(rg, pat, threads=threads))
            row.update(reference_s=tr, reference_threads=threads, equal=dev == ref)
        emit("exact_count", **row)

    # row 15: triangle_count
    td, dev = best(lambda: dg.triangle_count())
    tr, ref = once(lambda: R.triangle_count(rg))
    emit("triangle_count", graph=gname, device_s=td, reference_s=tr, reference_threads=1, count=dev,
         equal=dev == ref)

    # row 16: colour sparsification (colored_csr.cpp), c = 4
    td, (sub, cols, same) = best(lambda: dg.color_split(4, 7))
    tr, (rcols, _, _, rsame) = once(lambda: R.color_split(rg, 4, 7))
    emit("color_split", graph=gname, colors=4, device_s=td, reference_s=tr, reference_threads=1,
         same_color_edges=same, equal=bool(same == rsame and (cols == rcols).all()))

    # row 18: gs_estimate, colour scheme (gs_engine.cpp:42-75), 4-clique, c = 4
    plan = A.compile_plan("4clique")
    td, dev = best(lambda: A.gs_estimate(dg, plan, "color", colors=4, seed=11))
    tr, ref = once(lambda: R.gs_estimate(rg, "4clique", 1, colors=4, seed=11, threads=threads))
    emit("gs_estimate", graph=gname, pattern="4clique", scheme="color", colors=4, device_s=td, reference_s=tr,
         reference_threads=threads, raw_count=dev.raw_count, estimate=dev.estimate,
         equal=dev.raw_count == ref[1] and dev.estimate == ref[0])

    # row 17: Bernoulli sparsification p = 0.3 (device only: arc-for-arc parity is in the GPU suite)
    td, sub = best(lambda: dg.bernoulli_sparsify(0.3, 5))
    emit("bernoulli_sparsify", graph=gname, p=0.3, device_s=td, kept_edges=sub.info()["edge_count"])

    # rows 7 / 3b: online NS to 1 %@95 %, eager vs lazy (reference: workers = threads)
    for pat in ("triangle", "4clique"):
        for mode in ("eager", "lazy"):
            plan = A.compile_plan(pat, mode)
            pol = A.OnlinePolicy(max_samples=1 << 26)
            td, r = best(lambda: A.run_ns_online(dg, plan, 0.01, 0.05, pol, seed=1))
            row = dict(graph=gname, pattern=pat, verify=mode, device_s=td, n=r.report.n,
                       converged=bool(r.report.converged))
            if not (mode == "lazy" and pat != "triangle"):  # lazy 4-clique: ~2^26 reference samples, skipped
                tr, rr = once(lambda: R.ns_online(rg, pat, 0.01, 0.05, pol, 1, workers=1,
                                                  mode=0 if mode == "eager" else 1))
                row.update(reference_s=tr, reference_threads=1,
                           equal=(r.report.n == rr.report.n and r.accumulator.hits == rr.accumulator.hits))
            emit("ns_online", **row)

    # row 11b: device ingest vs the host builder (same algorithm as csr_graph.cpp:46-72)
    for s in ((16, 20) if quick else (20, 22)):
        td, dgi = best(lambda: A.rmat_device(s, 16, seed=1, relabel=True))
        th, hg = once(lambda: A.rmat(s, 16, seed=1).relabel_by_degree())
        emit("graph_ingest", graph=f"rmat{s}_ef16_relabelled", device_s=td, host_builder_s=th,
             edges=dgi.info()["edge_count"], equal=dgi.info()["edge_count"] == hg.edge_count)

    # row 22: dense/sparse split on the needle config (n = 2^22, 1000 planted K5), device only
    if not quick:
        nd = A.er_fast_device(1 << 22, (1 << 22) * 4, seed=4, planted_k=5, planted_count=1000)
        plan = A.compile_plan("5clique")
        td, res = best(lambda: A.region_split(nd, plan, 16, dense="exact"))
        te, exact = best(lambda: A.exact_count(nd, plan))
        emit("region_split", graph="er_n2^22_deg8_planted1000K5", pattern="5clique", device_s=td,
             exact_count_s=te, estimate=res.estimate, exact=exact, equal=res.estimate == exact)


if __name__ == "__main__":
    main()
