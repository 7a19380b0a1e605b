"""CPU: the C oracle restatement pinned against golden vectors of the compiled reference.

tests/golden/*.json come from the UNMODIFIED reference (tests/golden/make_golden.py
through oracle/_ref). Every check here is bit-exact except where noted.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from paper_2405_03488_b200._abi import Accumulator, OnlinePolicy

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def h64(*arrays):
    m = hashlib.sha256()
    for a in arrays:
        m.update(np.ascontiguousarray(a).tobytes())
    return m.hexdigest()[:32]


def test_rng_streams(oracle):
    """CounterRng / derive_key / Lemire next_below / next_double (rng.hpp:10-51)."""
    g = load("rng.json")
    for seed, s1, s2, key in g["derive_key"]:
        assert oracle.L.orc_derive_key(seed, s1, s2) == key
    for seed, s1, s2, seq in g["u64"]:
        assert oracle.rng_u64(seed, s1, s2, len(seq)).tolist() == seq
    for seed, s1, s2, seq in g["double"]:
        assert [float(x).hex() for x in oracle.rng_double(seed, s1, s2, len(seq))] == seq
    for seed, bound, seq in g["below"]:
        assert oracle.rng_below(seed, 0, 4, bound, len(seq)).tolist() == seq
    for seed, u, v, p, keep in g["edge_keep"]:
        assert oracle.L.orc_edge_keep(seed, u, v, p) == keep
    for seed, v, c, col in g["vertex_color"]:
        assert oracle.L.orc_vertex_color(seed, v, c) == col


def test_stats(oracle):
    """inv_norm_cdf and predicted_error (stats.cpp:14-70), bit-exact."""
    g = load("stats.json")
    for q, z in g["inv_norm_cdf"]:
        assert oracle.inv_norm_cdf(q).hex() == z
    for case in g["predicted_error"]:
        rep = oracle.predicted_error(Accumulator(*case["acc"]), case["delta"])
        assert rep.mu.hex() == case["mu"] and rep.sigma.hex() == case["sigma"]
        assert rep.epsilon_hat.hex() == case["epsilon_hat"] and rep.n == case["n"]
    with pytest.raises(ValueError):
        oracle.inv_norm_cdf(0.0)


def _er(agpm, n, p, seed):
    return agpm.er_graph(n, p, seed)


def test_draw_records(agpm, oracle):
    """Per-sample value/hit/bindings of draw_sample (ns_engine.cpp:27-53) on reference graphs."""
    g = load("samples.json")
    for key, rec in g.items():
        if key.startswith("config1"):
            continue
        _, n, p, sg, pat, seed, first = key.split("|")
        graph = _er(agpm, int(n), float(p), int(sg))
        off, nbr = graph.arrays()
        plan = agpm.compile_plan(pat)
        count = len(rec["values"])
        v, h, b = oracle.draw_records(off, nbr, graph.edge_count, plan, int(seed), int(first), count)
        assert [float(x).hex() for x in v] == rec["values"], key
        assert h.tolist() == rec["hits"], key
        assert b.tolist() == rec["bindings"], key


def test_lazy_draw_records_and_online(agpm, oracle):
    """Lazy verification (NS-base, walker.hpp:56-62 / 88-107): the oracle's records
    and online stop points equal the compiled reference's (samples_lazy.json)."""
    g = load("samples_lazy.json")
    for key, rec in g["records"].items():
        _, n, p, sg, pat, seed, first = key.split("|")
        graph = _er(agpm, int(n), float(p), int(sg))
        off, nbr = graph.arrays()
        plan = agpm.compile_plan(pat, "lazy")
        count = len(rec["values"])
        v, h, b = oracle.draw_records(off, nbr, graph.edge_count, plan, int(seed), int(first), count)
        assert [float(x).hex() for x in v] == rec["values"], key
        assert h.tolist() == rec["hits"], key
        assert b.tolist() == rec["bindings"], key
    for key, rec in g["online"].items():
        _, n, p, sg, pat, eps = key.split("|")
        graph = _er(agpm, int(n), float(p), int(sg))
        off, nbr = graph.arrays()
        r = oracle.ns_online(off, nbr, graph.edge_count, agpm.compile_plan(pat, "lazy"), float(eps), 0.05,
                             OnlinePolicy(1000, 10**7, 0), 3)
        assert (r.report.n, r.windows, r.accumulator.hits, r.report.converged) == \
            (rec["n"], rec["windows"], rec["hits"], rec["converged"]), key
        assert float(r.report.mu).hex() == rec["mu"], key


def test_config1_records_hash(agpm, oracle):
    """Config 1 (er_graph(10^4, 20/9999, 1), degree-relabelled), triangle, seed 1: the first
    2^16 sample records hash-equal the reference's."""
    rec = load("samples.json")["config1_relabelled|triangle|1|0|65536"]
    g = agpm.er_graph(10000, 20 / 9999, 1).relabel_by_degree()
    off, nbr = g.arrays()
    assert h64(off, nbr) == rec["graph_hash"]
    v, h, b = oracle.draw_records(off, nbr, g.edge_count, agpm.compile_plan("triangle"), 1, 0, 1 << 16)
    assert int(h.sum()) == rec["hits"]
    assert h64(v, h, b) == rec["records_hash"]


def test_exact_counts(agpm, oracle):
    """exact_count (exact_engine.cpp:66-91) incl. symmetry-off and oriented cliques."""
    g = load("counts.json")["exact"]
    ref_graphs = {
        "'complete'|5": [(i, j) for i in range(5) for j in range(i + 1, 5)],
        "'complete'|6": [(i, j) for i in range(6) for j in range(i + 1, 6)],
        "'cycle'|6": [(i, (i + 1) % 6) for i in range(6)],
        "'path'|6": [(i, i + 1) for i in range(5)],
        "'star'|5": [(0, i) for i in range(1, 6)],
    }
    for key, pats in g.items():
        if key.startswith("'er'"):
            _, n, p, s = key.split("|")
            graph = agpm.er_graph(int(n), float(p), int(s))
        else:
            nmin = int(key.split("|")[1]) + (1 if key.startswith("'star'") else 0)
            graph = agpm.CsrGraph.from_edges(ref_graphs[key], nmin)
        off, nbr = graph.arrays()
        for pat, res in pats.items():
            if pat == "oriented":
                og = graph.orient_by_degree()
                ooff, onbr = og.arrays()
                for cp, cnt in res.items():
                    assert oracle.exact_count(ooff, onbr, og.edge_count, agpm.compile_plan(cp), oriented=True) == cnt
                continue
            assert oracle.exact_count(off, nbr, graph.edge_count, agpm.compile_plan(pat)) == res["count"], (key, pat)
            nosym = agpm.compile_plan(pat, enable_symmetry=False)
            assert oracle.exact_count(off, nbr, graph.edge_count, nosym) == res["count_nosym"], (key, pat)
            if res["brute"] is not None:
                assert res["count"] == res["brute"]


def test_online_runs(agpm, oracle):
    """run_ns_online, workers = 1 (ns_engine.cpp:106-140): same stop n and bit-equal sums."""
    g = load("counts.json")["online"]
    for key, r in g.items():
        _, n, p, sg, pat, eps, delta, seed = key.split("|")
        graph = agpm.er_graph(int(n), float(p), int(sg))
        off, nbr = graph.arrays()
        res = oracle.ns_online(off, nbr, graph.edge_count, agpm.compile_plan(pat), float(eps), float(delta),
                               OnlinePolicy(), int(seed))
        assert res.report.n == r["n"] and res.windows == r["windows"] and res.accumulator.hits == r["hits"]
        assert res.accumulator.sum.hex() == r["sum"] and res.accumulator.squared_sum.hex() == r["squared_sum"]
        assert res.report.epsilon_hat.hex() == r["epsilon_hat"] and bool(res.report.converged) == r["converged"]


def test_color_split(agpm, oracle):
    """ColoredCsr::color_vertices + build_splits (colored_csr.cpp:14-54)."""
    g = load("counts.json")["split"]
    graph = agpm.er_graph(60, 0.2, 17)
    off, nbr = graph.arrays()
    for key, r in g.items():
        c, seed = map(int, key.split("|"))
        colors, split, out, same = oracle.color_split(off, nbr, c, seed)
        assert colors.tolist() == r["colors"] and split.tolist() == r["split_end"]
        assert h64(out) == r["nbr_hash"] and same == r["same_edges"]


def test_triangle_count(agpm, oracle):
    g = load("counts.json")["triangle_count"]
    for key, cnt in g.items():
        _, n, p, s = key.split("|")
        off, nbr = agpm.er_graph(int(n), float(p), int(s)).arrays()
        assert oracle.triangle_count(off, nbr) == cnt


def test_colored_exact_counts(agpm, oracle):
    """The GS inner count: exact_count on the colour-sparsified view (gs_engine.cpp:59-67)."""
    g = load("counts.json")["colored"]
    graph = agpm.er_graph(200, 0.08, 71)
    off, nbr = graph.arrays()
    for pat, per_c in g.items():
        for c, cnt in per_c.items():
            colors, split, pnbr, same = oracle.color_split(off, nbr, int(c), 7)
            got = oracle.exact_count(off[:-1], pnbr, same, agpm.compile_plan(pat), end=split)
            assert got == cnt, (pat, c)


# Philox4x32-10 known-answer vectors of the published algorithm (Salmon et al.,
# SC'11): counter / key -> the four output words after ten rounds.
PHILOX_KAT = [
    ([0, 0, 0, 0], (0, 0), [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
    ([0xFFFFFFFF] * 4, (0xFFFFFFFF, 0xFFFFFFFF), [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
    ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], (0xA4093822, 0x299F31D0),
     [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]),
]


@pytest.mark.parametrize("ctr,key,want", PHILOX_KAT)
def test_philox_known_answers(oracle, ctr, key, want):
    """The optional Philox stream's block function (oracle restatement; the
    device copy in csrc/rng.cuh is checked against this one record for record)."""
    assert oracle.philox4x32_10(ctr, key) == want


def test_philox_stream_unbiased(agpm, oracle):
    """Philox-stream NS is a valid estimator: on a small ER graph the mean of
    2^17 samples is within 5 sigma of the exact count (the draw procedure is the
    reference's; only the random numbers differ)."""
    import numpy as np

    g = agpm.er_graph(120, 0.15, 3)
    off, nbr = g.arrays()
    for pat in ("triangle", "4cycle"):
        plan = agpm.compile_plan(pat)
        exact = oracle.exact_count(off, nbr, g.edge_count, plan)
        v, h, b = oracle.draw_records_philox(off, nbr, g.edge_count, plan, 11, 0, 1 << 17)
        mu, sd = v.mean(), v.std() / np.sqrt(len(v))
        assert abs(mu - exact) <= 5 * sd, (pat, mu, exact, sd)
        cv, ch, cb = oracle.draw_records(off, nbr, g.edge_count, plan, 11, 0, 1 << 10)
        assert not np.array_equal(v[: 1 << 10], cv)  # a different stream


def test_multithreaded_checker_equals_sequential(agpm, oracle):
    """The parallel checker variants used by the big-config parity tests
    (orc_draw_records_mt, orc_ns_online_mt) give the sequential oracle's results
    bit for bit: records per sample id, online stop n, hits and the in-order sums."""
    g = agpm.rmat(11, 16, seed=5).relabel_by_degree()
    off, nbr = g.arrays()
    for spec in ("4clique", "4cycle", "triangle"):
        plan = agpm.compile_plan(spec)
        for first in (0, 1 << 40):
            a = oracle.draw_records(off, nbr, g.edge_count, plan, 3, first, 3000)
            b = oracle.draw_records_mt(off, nbr, g.edge_count, plan, 3, first, 3000, threads=4)
            for x, y in zip(a, b):
                assert np.array_equal(x, y), spec
        pol = OnlinePolicy()
        s = oracle.ns_online(off, nbr, g.edge_count, plan, 0.02, 0.05, pol, 7)
        p = oracle.ns_online_mt(off, nbr, g.edge_count, plan, 0.02, 0.05, pol, 7, threads=4)
        assert (s.report.n, s.windows, s.accumulator.hits) == (p.report.n, p.windows, p.accumulator.hits)
        assert s.accumulator.sum.hex() == p.accumulator.sum.hex()
        assert s.accumulator.squared_sum.hex() == p.accumulator.squared_sum.hex()
        assert s.report.epsilon_hat.hex() == p.report.epsilon_hat.hex()


def test_reference_arm_graph_equals_product_graph(agpm, ref):
    """bench.py's reference arm builds its RMAT input with no product code
    (oracle generator -> reference from_edges -> oracle relabel -> AGPM v1 ->
    reference load_graph_auto); it must be the product's graph array for array."""
    from oracle_bindings import reference_rmat_graph

    for scale, ef, seed in ((10, 16, 1), (13, 8, 5)):
        _, rg = reference_rmat_graph(scale, ef, seed=seed)
        off, nbr = rg.arrays()
        g = agpm.rmat(scale, ef, 0.57, 0.19, 0.19, seed=seed).relabel_by_degree()
        poff, pnbr = g.arrays()
        assert np.array_equal(off, poff) and np.array_equal(nbr, pnbr)
        assert rg.info()[1] == g.edge_count
