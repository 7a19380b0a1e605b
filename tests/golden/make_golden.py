#!/usr/bin/env python
"""Regenerate tests/golden/*.json from the UNMODIFIED reference.

Runs the reference library compiled from /root/reference/proj/src by
oracle/Makefile (oracle/_ref/libagpm_ref.so, behind oracle/ref_shim.cpp) and
records its outputs on seeded inputs: RNG streams, statistics, compiled plans,
generator outputs, per-sample draw records, exact / colour-sparsified counts,
online runs and colour splits. The CPU test suite pins the C oracle
restatement and the product's host logic against these files; the GPU suite
reuses them. Needs the reference tree (this container only):

    python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle_bindings import RefLib, build_oracle  # noqa: E402
from paper_2405_03488_b200._abi import OnlinePolicy  # noqa: E402


def h64(*arrays):
    m = hashlib.sha256()
    for a in arrays:
        m.update(np.ascontiguousarray(a).tobytes())
    return m.hexdigest()[:32]


def dump(name, obj):
    with open(os.path.join(HERE, name), "w") as f:
        json.dump(obj, f, indent=1, sort_keys=True)
    print("wrote", name)


BUILTINS = ["triangle", "4clique", "5clique", "6clique", "7clique", "8clique", "9clique", "4cycle", "5path",
            "house", "dumbbell", "3motif-wedge", "3motif-triangle", "4motif-path", "4motif-star", "4motif-cycle",
            "4motif-tailedtriangle", "4motif-diamond", "4motif-clique"]

# (n, p, seed) reference er_graph instances used across fixtures
ER_SMALL = [(7, 0.45, 321), (9, 0.35, 101), (12, 0.3, 500), (60, 0.2, 17), (100, 0.1, 66), (200, 0.08, 71)]


LAZY_CASES = [((200, 0.08, 71), "4clique", 9, 12345, 256), ((100, 0.1, 66), "triangle", 5, 0, 256),
              ((60, 0.2, 17), "4cycle", 3, 77, 256), ((60, 0.2, 17), "house", 3, 0, 256),
              ((60, 0.2, 17), "4motif-star", 8, 0, 256), ((100, 0.1, 66), "5path", 11, 500, 256),
              ((200, 0.08, 71), "dumbbell", 2, 0, 128), ((60, 0.2, 17), "4motif-diamond", 4, 9, 256),
              ((60, 0.2, 17), "5clique", 6, 0, 256)]


def lazy_records(R):
    """Lazy-verify (NS-base) draw records and online runs (ns_engine.cpp:27-53, 106-140)."""
    out = {"records": {}, "online": {}}
    for (n, p, seed_g), pat, seed, first, count in LAZY_CASES:
        g = R.er_graph(n, p, seed_g)
        v, h, b = R.draw_records(g, pat, seed, first, count, mode=1)
        out["records"][f"er|{n}|{p!r}|{seed_g}|{pat}|{seed}|{first}"] = {
            "values": [float(x).hex() for x in v], "hits": h.tolist(), "bindings": b.tolist()}
    for (n, p, seed_g), pat, eps in [((200, 0.08, 71), "triangle", 0.05), ((200, 0.08, 71), "4cycle", 0.1)]:
        g = R.er_graph(n, p, seed_g)
        r = R.ns_online(g, pat, eps, 0.05, OnlinePolicy(1000, 10**7, 0), 3, mode=1)
        out["online"][f"er|{n}|{p!r}|{seed_g}|{pat}|{eps!r}"] = {
            "n": r.report.n, "windows": r.windows, "hits": r.accumulator.hits, "mu": float(r.report.mu).hex(),
            "converged": r.report.converged}
    dump("samples_lazy.json", out)


def main():
    build_oracle(ref=True)
    R = RefLib()
    if sys.argv[1:] == ["lazy"]:
        lazy_records(R)
        return
    lazy_records(R)

    # ---------------------------------------------------------------- rng (rng.hpp)
    rng = {"derive_key": [], "u64": [], "below": [], "double": [], "edge_keep": [], "vertex_color": []}
    for seed, s1, s2 in [(0, 0, 0), (1, 0, 0), (1, 0, 12345), (42, 7, 99), (2**63 + 5, 2**40, 2**33 + 1)]:
        rng["derive_key"].append([seed, s1, s2, int(R.L.ref_derive_key(seed, s1, s2))])
        out = np.zeros(16, np.uint64)
        R.L.ref_rng_u64(seed, s1, s2, 16, out.ctypes.data_as(R.L.ref_rng_u64.argtypes[4]))
        rng["u64"].append([seed, s1, s2, [int(x) for x in out]])
        d = np.zeros(8, np.float64)
        R.L.ref_rng_double(seed, s1, s2, 8, d.ctypes.data_as(R.L.ref_rng_double.argtypes[4]))
        rng["double"].append([seed, s1, s2, [float(x).hex() for x in d]])
    # bounds include near-2^64 values where Lemire rejection fires often
    for seed, bound in [(3, 1), (3, 2), (5, 7), (9, 1000), (11, 2**31 + 11), (13, 2**63 + 3), (17, 2**64 - 3),
                        (19, 3 * 2**62 + 1)]:
        out = np.zeros(32, np.uint64)
        R.L.ref_rng_below(seed, 0, 4, bound, 32, out.ctypes.data_as(R.L.ref_rng_below.argtypes[5]))
        rng["below"].append([seed, bound, [int(x) for x in out]])
    for seed, u, v, p in [(1, 0, 1, 0.5), (1, 9, 3, 0.5), (77, 123456, 7, 0.1), (5, 2**31, 2**31 + 1, 0.9)]:
        rng["edge_keep"].append([seed, u, v, p, int(R.L.ref_edge_keep(seed, u, v, p))])
    for seed, v, c in [(1, 0, 4), (1, 17, 4), (9, 123, 3), (2**40, 99999, 18), (7, 5, 1)]:
        rng["vertex_color"].append([seed, v, c, int(R.L.ref_vertex_color(seed, v, c))])
    dump("rng.json", rng)

    # ---------------------------------------------------------------- stats (stats.cpp)
    import ctypes as C
    from paper_2405_03488_b200._abi import Accumulator, Report
    stats = {"inv_norm_cdf": [], "predicted_error": []}
    for q in [0.001, 0.01, 0.02425, 0.025, 0.1, 0.5, 0.9, 0.975, 0.995, 0.999]:
        out = C.c_double()
        R.L.ref_inv_norm_cdf(q, C.byref(out))
        stats["inv_norm_cdf"].append([q, out.value.hex()])
    for acc, delta in [((4, 4, 8.0, 16.0), 0.05), ((2, 1, 4.0, 16.0), 0.05), ((100, 0, 0.0, 0.0), 0.05),
                       ((1, 1, 5.0, 25.0), 0.05), ((1000, 300, 12345.5, 987654.25), 0.01),
                       ((5000, 2000, 21000.0, 221000.0), 0.1)]:
        a = Accumulator(*acc)
        rep = Report()
        R.L.ref_predicted_error(C.byref(a), delta, C.byref(rep))
        stats["predicted_error"].append({"acc": list(acc), "delta": delta, "mu": rep.mu.hex(),
                                         "sigma": rep.sigma.hex(), "epsilon_hat": rep.epsilon_hat.hex(),
                                         "n": rep.n, "hit_rate": rep.hit_rate.hex()})
    dump("stats.json", stats)

    # ---------------------------------------------------------------- plans (plan.cpp)
    plans = {}
    for name in BUILTINS:
        for mode in (0, 1):
            for sym in (1, 0):
                for ind in ("", "edge", "vertex"):
                    key = f"{name}|{mode}|{sym}|{ind}"
                    plans[key] = {"plan": R.plan(name, mode, bool(sym), ind).to_dict(),
                                  "rule": R.scaling_rule(name, mode, bool(sym), ind)}
    customs = ["custom:4:0-1,1-2,2-3,3-0", "custom:3:0-1,1-2", "custom:5:0-1,1-2,2-3,3-4,4-0,0-2",
               "custom:6:0-1,0-2,0-3,0-4,0-5", "custom:4:0-1,0-2,0-3,1-2"]
    for spec in customs:
        for mode in (0, 1):
            key = f"{spec}|{mode}|1|"
            plans[key] = {"plan": R.plan(spec, mode, True, "").to_dict(), "rule": R.scaling_rule(spec, mode)}
    errors = {}
    for spec, ind in [("custom:4:0-1", ""), ("custom:3:0-0,1-2", ""), ("custom:3:0-9", ""),
                      ("triangle", "sideways"), ("pentagon", ""), ("custom:x:0-1", ""), ("custom:3:0-1,12", ""),
                      ("custom:3:a-1", ""), ("custom:1:", ""), ("custom:10:0-1", ""), ("custom:3", "")]:
        st, msg = R.plan_error(spec, 0, True, ind)
        errors[f"{spec}|{ind}"] = [st, msg]
    auts = {n: R.automorphism_count(n) for n in BUILTINS}
    dump("plans.json", {"plans": plans, "errors": errors, "automorphisms": auts})

    # ---------------------------------------------------------------- graphs + generators
    graphs = {}
    for n, p, seed in ER_SMALL + [(10000, 20 / 9999, 1)]:
        g = R.er_graph(n, p, seed)
        off, nbr = g.arrays()
        _, m, arcs, _ = g.info()
        graphs[f"er|{n}|{p!r}|{seed}"] = {"m": m, "arcs": arcs, "hash": h64(off, nbr)}
    rnd = np.random.default_rng(99).integers(0, 30, size=(100, 2)).astype(np.uint32)
    g = R.from_edges(rnd)
    off, nbr = g.arrays()
    graphs["from_edges|random30"] = {"edges": rnd.tolist(), "m": g.info()[1], "hash": h64(off, nbr)}
    dump("graphs.json", graphs)

    # ---------------------------------------------------------------- per-sample records (ns_engine.cpp:27-53)
    samples = {}
    cases = [((200, 0.08, 71), "4clique", 9, 12345, 256), ((100, 0.1, 66), "triangle", 5, 0, 256),
             ((60, 0.2, 17), "4cycle", 3, 77, 256), ((60, 0.2, 17), "house", 3, 0, 256),
             ((60, 0.2, 17), "4motif-path", 8, 0, 256), ((100, 0.1, 66), "5path", 11, 500, 256),
             ((200, 0.08, 71), "dumbbell", 2, 0, 128)]
    for (n, p, seed_g), pat, seed, first, count in cases:
        g = R.er_graph(n, p, seed_g)
        v, h, b = R.draw_records(g, pat, seed, first, count)
        samples[f"er|{n}|{p!r}|{seed_g}|{pat}|{seed}|{first}"] = {
            "values": [float(x).hex() for x in v], "hits": h.tolist(), "bindings": b.tolist()}
    # config 1 graph (er_graph(10^4, 20/9999, 1)) relabelled by (degree, id): first 2^16 samples, hashed
    g = R.er_graph(10000, 20 / 9999, 1)
    off, nbr = g.arrays()
    deg = np.diff(off)
    order = np.lexsort((np.arange(len(deg)), deg))
    new_id = np.empty_like(order)
    new_id[order] = np.arange(len(order))
    edges = []
    for u in range(len(deg)):
        for w in nbr[off[u]:off[u + 1]]:
            if u < w:
                edges.append((new_id[u], new_id[w]))
    gr = R.from_edges(np.array(edges, np.uint32), len(deg))
    roff, rnbr = gr.arrays()
    v, h, b = R.draw_records(gr, "triangle", 1, 0, 1 << 16)
    samples["config1_relabelled|triangle|1|0|65536"] = {
        "graph_hash": h64(roff, rnbr), "records_hash": h64(v, h, b), "hits": int(h.sum()),
        "first": {"values": [float(x).hex() for x in v[:64]], "bindings": b[:64].tolist()}}
    dump("samples.json", samples)

    # ---------------------------------------------------------------- exact / colour / online / split
    exact = {}
    small = [("complete", 5), ("complete", 6), ("cycle", 6), ("path", 6), ("star", 5)] + [("er",) + t for t in ER_SMALL[:4]]
    for spec in small:
        if spec[0] == "er":
            g = R.er_graph(*spec[1:])
        else:
            g = getattr(R, spec[0])(spec[1])
        key = "|".join(map(repr, spec))
        exact[key] = {}
        for pat in BUILTINS[:3] + BUILTINS[7:]:
            exact[key][pat] = {"count": R.exact_count(g, pat),
                               "count_nosym": R.exact_count(g, pat, sym=False),
                               "brute": R.brute_force(g, pat) if g.info()[0] <= 14 else None}
        og = R.orient(g)
        exact[key]["oriented"] = {pat: R.exact_count(og, pat) for pat in ["triangle", "4clique", "5clique"]}
    g = R.er_graph(200, 0.08, 71)
    colored = {pat: {str(c): R.exact_count_colored(g, pat, c, 7) for c in (1, 2, 4)} for pat in
               ["triangle", "4clique", "4cycle", "house"]}
    gs = {}
    for pat in ["triangle", "4cycle"]:
        gs[pat] = {"color4": list(R.gs_estimate(g, pat, 1, colors=4, seed=11)),
                   "bern05": list(R.gs_estimate(g, pat, 0, p=0.5, seed=11))}
    online = {}
    for (n, p, sg), pat, eps, delta, seed in [((200, 0.08, 71), "4clique", 0.2, 0.05, 31),
                                              ((100, 0.1, 66), "triangle", 0.05, 0.05, 3),
                                              ((200, 0.08, 71), "4cycle", 0.05, 0.01, 8)]:
        g = R.er_graph(n, p, sg)
        r = R.ns_online(g, pat, eps, delta, OnlinePolicy(), seed)
        online[f"er|{n}|{p!r}|{sg}|{pat}|{eps}|{delta}|{seed}"] = {
            "n": r.report.n, "windows": r.windows, "hits": r.accumulator.hits, "sum": r.accumulator.sum.hex(),
            "squared_sum": r.accumulator.squared_sum.hex(), "converged": r.report.converged,
            "epsilon_hat": r.report.epsilon_hat.hex(), "mu": r.report.mu.hex()}
    g = R.er_graph(60, 0.2, 17)
    split = {}
    for c, seed in [(2, 5), (3, 9), (4, 19)]:
        colors, se, nb, same = R.color_split(g, c, seed)
        split[f"{c}|{seed}"] = {"colors": colors.tolist(), "split_end": se.tolist(), "nbr_hash": h64(nb),
                                "same_edges": same}
    tri = {f"er|{n}|{p!r}|{s}": R.triangle_count(R.er_graph(n, p, s)) for n, p, s in ER_SMALL}
    dump("counts.json", {"exact": exact, "colored": colored, "gs": gs, "online": online, "split": split,
                         "triangle_count": tri})


if __name__ == "__main__":
    main()
