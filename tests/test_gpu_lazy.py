"""GPU parity for lazy-verify neighbour sampling (NS-base, ns_lazy.cu).

Per-sample values, hits and bindings of the device lazy sampler equal the
oracle's (itself pinned to the compiled reference by samples_lazy.json):
candidate set = union of the bound vertices' lists minus bound vertices
(walker.hpp:56-62), tree-parent check after each pick (ns_engine.cpp:41-46),
closure / terminal / induced checks at the end (walker.hpp:88-107).
"""
import json
import os

import numpy as np
import pytest

from paper_2405_03488_b200._abi import OnlinePolicy

pytestmark = pytest.mark.gpu

PATTERNS = ["triangle", "4clique", "5clique", "4cycle", "house", "5path", "dumbbell", "6clique",
            "3motif-wedge", "4motif-path", "4motif-star", "4motif-diamond", "4motif-tailedtriangle",
            "4motif-cycle", "3motif-triangle", "4motif-clique"]


@pytest.fixture(scope="module")
def graphs(agpm):
    return {
        "er200": agpm.er_graph(200, 0.08, 71),
        "er60_dense_rel": agpm.er_graph(60, 0.5, 5).relabel_by_degree(),
        "rmat10_rel": agpm.rmat(10, 8, seed=3).relabel_by_degree(),
        "star": agpm.CsrGraph.from_edges([[0, i] for i in range(1, 70)] + [[1, 2], [3, 4]]),
    }


@pytest.mark.parametrize("name", ["er200", "er60_dense_rel", "rmat10_rel", "star"])
@pytest.mark.parametrize("pattern", PATTERNS)
def test_lazy_draw_bit_exact(agpm, oracle, graphs, name, pattern):
    g = graphs[name]
    off, nbr = g.arrays()
    plan = agpm.compile_plan(pattern, "lazy")
    dg = agpm.DeviceGraph(g)
    count = 3000 if plan.k <= 5 else 1000
    v, h, b = agpm.draw_samples(dg, plan, 9, 777, count)
    ov, oh, ob = oracle.draw_records(off, nbr, g.edge_count, plan, 9, 777, count)
    np.testing.assert_array_equal(h, oh)
    np.testing.assert_array_equal(v, ov)
    np.testing.assert_array_equal(b, ob)


def test_lazy_golden_records(agpm):
    """Device lazy records == the compiled reference's (tests/golden/samples_lazy.json)."""
    with open(os.path.join(os.path.dirname(__file__), "golden", "samples_lazy.json")) as f:
        g = json.load(f)
    for key, rec in g["records"].items():
        _, n, p, sg, pat, seed, first = key.split("|")
        graph = agpm.er_graph(int(n), float(p), int(sg))
        v, h, b = agpm.draw_samples(agpm.DeviceGraph(graph), agpm.compile_plan(pat, "lazy"), int(seed),
                                    int(first), len(rec["values"]))
        assert [float(x).hex() for x in v] == rec["values"], key
        assert h.tolist() == rec["hits"], key
        assert b.tolist() == rec["bindings"], key
    for key, rec in g["online"].items():
        _, n, p, sg, pat, eps = key.split("|")
        graph = agpm.er_graph(int(n), float(p), int(sg))
        r = agpm.run_ns_online(agpm.DeviceGraph(graph), agpm.compile_plan(pat, "lazy"), float(eps), 0.05,
                               OnlinePolicy(1000, 10**7, 0), seed=3)
        assert (r.report.n, r.windows, r.accumulator.hits) == (rec["n"], rec["windows"], rec["hits"]), key
        assert abs(r.report.mu - float.fromhex(rec["mu"])) <= 1e-12 * abs(float.fromhex(rec["mu"]))


def test_lazy_fixed_budget_and_unbiased(agpm, oracle):
    g = agpm.rmat(11, 16, seed=5).relabel_by_degree()
    off, nbr = g.arrays()
    dg = agpm.DeviceGraph(g)
    plan = agpm.compile_plan("triangle", "lazy")
    acc = agpm.run_fixed_budget(dg, plan, 200000, 4)
    o = oracle.fixed_budget(off, nbr, g.edge_count, plan, 200000, 4)
    assert acc.n == o.n and acc.hits == o.hits
    assert abs(acc.sum - o.sum) <= 1e-12 * o.sum
    exact = agpm.exact_count(dg, agpm.compile_plan("triangle"))
    # both verification modes estimate the same count
    eager = agpm.run_fixed_budget(dg, agpm.compile_plan("triangle"), 200000, 4)
    assert abs(eager.sum / eager.n - exact) < 0.05 * exact
    assert abs(acc.sum / acc.n - exact) < 0.25 * exact


def test_lazy_bmin_rejected(agpm):
    g = agpm.er_graph(60, 0.2, 17)
    with pytest.raises(ValueError):
        agpm.bmin_bytes(agpm.DeviceGraph(g), agpm.compile_plan("triangle", "lazy"), 1, 0, 1000)
