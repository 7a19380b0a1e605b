"""GPU parity for the eager-verify sampler.

The CUDA path (through the C-ABI) against the C oracle restatement on the same
seeded inputs: per-sample value, hit AND matching-order bindings must be
bit-identical to the reference's draw_sample with stream CounterRng(seed, 0, id)
(ns_engine.cpp:27-53); accumulators agree exactly in n/hits and to
reduction-order rounding (relative 1e-12, the oracle's own streaming
tolerance is 1e-9, acceptance_main.cpp:413) in sum / squared sum; the online
run stops at the same n (ns_engine.cpp:106-140).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

PATTERNS = ["triangle", "4clique", "5clique", "4cycle", "house", "5path", "dumbbell", "6clique",
            "3motif-wedge", "4motif-path", "4motif-star", "4motif-diamond", "4motif-tailedtriangle",
            "4motif-cycle", "3motif-triangle", "4motif-clique"]


def _graphs(agpm):
    # small ER graphs (reference generator) plain and degree-relabelled, a
    # skewed RMAT graph whose hubs exercise the warp-cooperative path
    out = {
        "er200": agpm.er_graph(200, 0.08, 71),
        "er200_rel": agpm.er_graph(200, 0.08, 71).relabel_by_degree(),
        "er60_dense": agpm.er_graph(60, 0.5, 5).relabel_by_degree(),
        "rmat12_rel": agpm.rmat(12, 16, seed=3).relabel_by_degree(),
        "rmat12": agpm.rmat(12, 16, seed=3),
    }
    return out


@pytest.fixture(scope="module")
def graphs(agpm):
    return _graphs(agpm)


@pytest.fixture(params=["warp", "lane", "frontier", "frontier_reuse", "frontier_nocore", "flat",
                        "flat_nocore", "flat_core96", "frontier_core96"])
def strategy(agpm, request):
    agpm.set_strategy(request.param.split("_")[0])
    agpm.set_frontier_reuse(request.param == "frontier_reuse")
    # frontier: the dense-core bit matrix covers every vertex of the small test
    # graphs by default; "nocore" runs the splitter-search path instead and
    # "core96" a core of the top 96 ids only (mixed fast / generic samples)
    agpm.set_core_dim(0 if request.param.endswith("nocore") else 96 if request.param.endswith("core96") else 65536)
    yield request.param
    agpm.set_strategy("auto")
    agpm.set_frontier_reuse(False)
    agpm.set_core_dim(None)


@pytest.mark.parametrize("name", ["er200", "er200_rel", "er60_dense", "rmat12_rel", "rmat12"])
@pytest.mark.parametrize("pattern", PATTERNS)
def test_draw_bit_exact(agpm, oracle, graphs, name, pattern, strategy):
    g = graphs[name]
    off, nbr = g.arrays()
    m = g.edge_count
    plan = agpm.compile_plan(pattern, "eager")
    dg = agpm.DeviceGraph(g)
    count = 6000 if plan.k <= 5 else 2500
    first = 12345
    v, h, b = agpm.draw_samples(dg, plan, 9, first, count)
    ov, oh, ob = oracle.draw_records(off, nbr, m, plan, 9, first, count)
    np.testing.assert_array_equal(h, oh)
    np.testing.assert_array_equal(v, ov)  # bit-exact doubles
    np.testing.assert_array_equal(b, ob)


@pytest.mark.parametrize("relabel", [False, True])
@pytest.mark.parametrize("pattern", ["triangle", "4clique", "4cycle", "house", "4motif-diamond"])
@pytest.mark.parametrize("strat", ["flat", "flat_nocore", "frontier"])
def test_long_drivers_bit_exact(agpm, oracle, pattern, relabel, strat):
    """RMAT-16 hubs (degree > 2048): drivers longer than the flat sampler's
    round capacity take its warp-per-sample path; values and bindings still
    match the oracle record for record."""
    g = agpm.rmat(16, 16, seed=5)
    if relabel:
        g = g.relabel_by_degree()
    assert g.max_degree() > 4096
    off, nbr = g.arrays()
    plan = agpm.compile_plan(pattern)
    dg = agpm.DeviceGraph(g)
    agpm.set_strategy(strat.split("_")[0])
    agpm.set_core_dim(0 if strat.endswith("nocore") else 65536)
    try:
        v, h, b = agpm.draw_samples(dg, plan, 4, 777, 20000)
    finally:
        agpm.set_strategy("auto")
        agpm.set_core_dim(None)
    ov, oh, ob = oracle.draw_records(off, nbr, g.edge_count, plan, 4, 777, 20000)
    np.testing.assert_array_equal(v, ov)
    np.testing.assert_array_equal(b, ob)


def test_config1_first_2pow16_bit_exact(agpm, oracle, strategy):
    """Config 1 graph (er_graph(10^4, 20/9999, 1), degree-relabelled), triangle,
    stream seed 1: the first 2^16 samples match record for record."""
    g = agpm.er_graph(10000, 20 / 9999, 1).relabel_by_degree()
    off, nbr = g.arrays()
    plan = agpm.compile_plan("triangle")
    dg = agpm.DeviceGraph(g)
    v, h, b = agpm.draw_samples(dg, plan, 1, 0, 1 << 16)
    ov, oh, ob = oracle.draw_records(off, nbr, g.edge_count, plan, 1, 0, 1 << 16)
    np.testing.assert_array_equal(v, ov)
    np.testing.assert_array_equal(b, ob)


def test_fixed_budget_matches_oracle(agpm, oracle, strategy):
    g = agpm.rmat(11, 16, seed=5).relabel_by_degree()
    off, nbr = g.arrays()
    plan = agpm.compile_plan("4clique")
    dg = agpm.DeviceGraph(g)
    acc = agpm.run_fixed_budget(dg, plan, 200000, 77)
    o = oracle.fixed_budget(off, nbr, g.edge_count, plan, 200000, 77)
    assert acc.n == o.n and acc.hits == o.hits
    assert abs(acc.sum - o.sum) <= 1e-12 * abs(o.sum)
    assert abs(acc.squared_sum - o.squared_sum) <= 1e-12 * abs(o.squared_sum)


@pytest.mark.parametrize("pattern,eps", [("4clique", 0.05), ("triangle", 0.02), ("4cycle", 0.05)])
def test_online_stops_where_oracle_stops(agpm, oracle, pattern, eps, strategy):
    g = agpm.rmat(11, 16, seed=7).relabel_by_degree()
    off, nbr = g.arrays()
    plan = agpm.compile_plan(pattern)
    dg = agpm.DeviceGraph(g)
    pol = agpm.OnlinePolicy()
    r = agpm.run_ns_online(dg, plan, eps, 0.05, pol, seed=31)
    o = oracle.ns_online(off, nbr, g.edge_count, plan, eps, 0.05, pol, 31)
    assert r.report.converged == o.report.converged == 1
    assert r.report.n == o.report.n and r.windows == o.windows
    assert r.accumulator.hits == o.accumulator.hits
    assert abs(r.report.mu - o.report.mu) <= 1e-12 * o.report.mu
    assert abs(r.report.epsilon_hat - o.report.epsilon_hat) <= 1e-9 * o.report.epsilon_hat


def test_online_cap_without_matches(agpm):
    """Star graph has no triangle: the cap stops the run unconverged (test_ns_engine.cpp:148-158)."""
    star = agpm.CsrGraph.from_edges([[0, i] for i in range(1, 5)], 5)
    dg = agpm.DeviceGraph(star)
    plan = agpm.compile_plan("triangle")
    r = agpm.run_ns_online(dg, plan, 0.1, 0.01, agpm.OnlinePolicy(max_samples=5000), seed=3)
    assert not r.report.converged
    assert r.report.n == 5000 and r.accumulator.hits == 0
    assert np.isinf(r.report.epsilon_hat)


def test_t3_hits_with_scale_3(agpm):
    """draw_sample on T3 hits with value 3 about 1/3 of the time (test_ns_engine.cpp:73-90)."""
    tri = agpm.CsrGraph.from_edges([[0, 1], [1, 2], [0, 2]], 3)
    dg = agpm.DeviceGraph(tri)
    v, h, _ = agpm.draw_samples(dg, agpm.compile_plan("triangle"), 10, 0, 3000)
    assert set(np.unique(v)) <= {0.0, 3.0}
    assert abs(h.mean() - 1 / 3) < 0.05


def test_errors_are_loud(agpm):
    tri = agpm.CsrGraph.from_edges([[0, 1], [1, 2], [0, 2]], 3)
    dg = agpm.DeviceGraph(tri)
    with pytest.raises(ValueError):
        agpm.run_ns_online(dg, agpm.compile_plan("triangle"), 1.5, 0.05)
    empty = agpm.CsrGraph.from_edges(np.zeros((0, 2), np.uint32), 4)
    with pytest.raises(ValueError):
        agpm.draw_samples(agpm.DeviceGraph(empty), agpm.compile_plan("triangle"), 1, 0, 10)
    oriented = agpm.DeviceGraph(tri.orient_by_degree())
    with pytest.raises(ValueError):
        agpm.draw_samples(oriented, agpm.compile_plan("triangle"), 1, 0, 10)


@pytest.mark.parametrize("pattern", ["triangle", "4clique", "5clique", "4cycle", "house", "4motif-diamond", "dumbbell"])
def test_values_without_bindings(agpm, oracle, graphs, pattern, strategy):
    """Without bindings the frontier sampler only counts the last step's
    candidates (no pick): values must still equal the oracle's bit for bit."""
    g = graphs["rmat12_rel"]
    off, nbr = g.arrays()
    plan = agpm.compile_plan(pattern)
    v, h, _ = agpm.draw_samples(agpm.DeviceGraph(g), plan, 4, 999, 5000, with_bindings=False)
    ov, oh, _ = oracle.draw_records(off, nbr, g.edge_count, plan, 4, 999, 5000)
    np.testing.assert_array_equal(v, ov)


@pytest.mark.parametrize("pattern", ["7clique", "8clique", "9clique"])
@pytest.mark.parametrize("strat", ["flat", "frontier", "warp"])
def test_large_k_bit_exact(agpm, oracle, pattern, strat):
    """k = 7..9 instantiations (the register-capped flat kernels spill most
    there) on a dense graph where deep cliques are common: values, hits and
    bindings match the oracle record for record."""
    g = agpm.er_graph(48, 0.7, 13).relabel_by_degree()
    off, nbr = g.arrays()
    plan = agpm.compile_plan(pattern)
    dg = agpm.DeviceGraph(g)
    agpm.set_strategy(strat)
    try:
        v, h, b = agpm.draw_samples(dg, plan, 3, 99, 3000)
    finally:
        agpm.set_strategy("auto")
    ov, oh, ob = oracle.draw_records(off, nbr, g.edge_count, plan, 3, 99, 3000)
    assert np.count_nonzero(oh) > 0
    np.testing.assert_array_equal(v, ov)
    np.testing.assert_array_equal(b, ob)


@pytest.mark.parametrize("name", ["er200_rel", "er60_dense", "rmat12_rel", "rmat12"])
@pytest.mark.parametrize("pattern", ["triangle", "4clique", "5clique", "4cycle", "house", "4motif-diamond"])
def test_philox_stream_bit_exact(agpm, oracle, graphs, name, pattern):
    """Optional Philox4x32-10 stream (agpm_ns_set_rng(1), flat sampler): the
    device's per-sample values, hits and bindings equal the oracle's Philox
    restatement (whose block function passes the published known answers,
    tests/test_cpu_oracle.py)."""
    g = graphs[name]
    off, nbr = g.arrays()
    plan = agpm.compile_plan(pattern)
    dg = agpm.DeviceGraph(g)
    agpm.set_rng("philox")
    try:
        v, h, b = agpm.draw_samples(dg, plan, 21, 5000, 6000)
    finally:
        agpm.set_rng("counter")
    ov, oh, ob = oracle.draw_records_philox(off, nbr, g.edge_count, plan, 21, 5000, 6000)
    np.testing.assert_array_equal(v, ov)
    np.testing.assert_array_equal(b, ob)


def test_philox_policy_errors_and_estimate(agpm, oracle):
    g = agpm.er_graph(10000, 20 / 9999, 1).relabel_by_degree()  # config 1
    off, nbr = g.arrays()
    dg = agpm.DeviceGraph(g)
    plan = agpm.compile_plan("triangle")
    exact = agpm.exact_count(dg, plan)
    agpm.set_rng("philox")
    try:
        r = agpm.run_ns_online(dg, plan, 0.01, 0.05, agpm.OnlinePolicy(), seed=3)
        assert r.report.converged and abs(r.report.mu - exact) / exact < 0.03  # 3x the 1 % bound
        agpm.set_strategy("frontier")
        with pytest.raises(ValueError):
            agpm.draw_samples(dg, plan, 1, 0, 100)
        agpm.set_strategy("auto")
        with pytest.raises(ValueError):
            agpm.draw_samples(dg, agpm.compile_plan("triangle", "lazy"), 1, 0, 100)
    finally:
        agpm.set_rng("counter")
        agpm.set_strategy("auto")
    with pytest.raises(ValueError):
        agpm.set_rng("mt19937")


@pytest.mark.parametrize("strat", ["flat", "frontier"])
@pytest.mark.parametrize("pattern", ["triangle", "4clique", "5clique", "4cycle", "house"])
def test_twin_arc_hints_same_samples(agpm, oracle, graphs, strat, pattern):
    """The twin-arc index is built once as many ids as the view has arcs have been
    sampled on it and only changes search hints: the launches before (without)
    and after (with) draw the same records, equal to the oracle's."""
    for name in ("rmat12_rel", "rmat12", "er200_rel"):
        g = graphs[name]
        off, nbr = g.arrays()
        plan = agpm.compile_plan(pattern)
        dg = agpm.DeviceGraph(g)
        agpm.set_strategy(strat)
        try:
            arcs = dg.info()["arcs"]
            count = max(5000, (arcs + 1) // 2)  # two launches reach the view's arc count
            runs, sizes = [], []
            for _ in range(4):
                runs.append(agpm.draw_samples(dg, plan, 5, 300, count)[:3])
                sizes.append(dg.info()["device_bytes"])
        finally:
            agpm.set_strategy("auto")
        # the index really exists (4 B per arc) from the first launch that starts with
        # >= arcs ids already sampled on the view, and only from then on
        first_with = next(k for k in range(4) if k * count >= arcs)
        assert 1 <= first_with <= 3
        grow = [sizes[k] - sizes[k - 1] for k in range(1, 4)]
        assert grow == [4 * arcs if k == first_with else 0 for k in range(1, 4)]
        runs = [tuple(a[:5000] for a in r) for r in runs]
        ov, oh, ob = oracle.draw_records(off, nbr, g.edge_count, plan, 5, 300, 5000)
        for v, h, b in runs:
            np.testing.assert_array_equal(v, ov)
            np.testing.assert_array_equal(b, ob)


@pytest.mark.parametrize("pattern", ["triangle", "4cycle", "4clique", "5clique", "custom:5:0-1,0-2,1-2,2-3,2-4,3-4"])
@pytest.mark.parametrize("rng", ["counter", "philox"])
def test_flat_sorted_order_same_records(agpm, oracle, pattern, rng):
    """Launches of >= 2^20 ids run the flat
    sampler in seed-sorted processing order (ns_flat.cu: flat_order); values, hits
    and bindings are written by id, so the records equal the oracle's, and the same
    ids drawn in smaller (id-ordered) launches."""
    g = agpm.rmat(14, 16, seed=5).relabel_by_degree()
    off, nbr = g.arrays()
    plan = agpm.compile_plan(pattern)
    dg = agpm.DeviceGraph(g)
    first, count = (1 << 33) + 12345, (1 << 20) + 77
    agpm.set_strategy("flat")
    agpm.set_rng(rng)
    try:
        v, h, b = agpm.draw_samples(dg, plan, 9, first, count)[:3]
        parts = [agpm.draw_samples(dg, plan, 9, first + o, min(1 << 18, count - o))[:3]
                 for o in range(0, count, 1 << 18)]
    finally:
        agpm.set_strategy("auto")
        agpm.set_rng("counter")
    np.testing.assert_array_equal(v.view(np.uint64), np.concatenate([p[0] for p in parts]).view(np.uint64))
    np.testing.assert_array_equal(h, np.concatenate([p[1] for p in parts]))
    np.testing.assert_array_equal(b, np.concatenate([p[2] for p in parts]))
    assert int(h.sum()) > 0
    if rng == "counter":  # the reference stream: the oracle's records
        ov, oh, ob = oracle.draw_records_mt(off, nbr, g.edge_count, plan, 9, first, count)
        np.testing.assert_array_equal(v.view(np.uint64), ov.view(np.uint64))
        np.testing.assert_array_equal(h, oh)
        np.testing.assert_array_equal(b, ob)


def test_prepare_builds_indexes_same_samples(agpm, oracle, graphs):
    """agpm_graph_prepare builds the dense core and twin arcs eagerly: the view
    grows by the twin index at once and draws the oracle's records from its
    first launch on."""
    g = graphs["rmat12_rel"]
    off, nbr = g.arrays()
    dg = agpm.DeviceGraph(g)
    before = dg.info()["device_bytes"]
    dg.prepare()
    grown = dg.info()["device_bytes"] - before
    assert grown >= 4 * dg.info()["arcs"]  # twin arcs (+ the dense-core rows)
    plan = agpm.compile_plan("4clique")
    v, h, b = agpm.draw_samples(dg, plan, 3, 77, 1 << 18)
    ov, oh, ob = oracle.draw_records(off, nbr, g.edge_count, plan, 3, 77, 1 << 18)
    np.testing.assert_array_equal(v, ov)
    np.testing.assert_array_equal(b, ob)
    assert dg.info()["device_bytes"] - before == grown  # nothing rebuilt on launch


def test_self_loops_rejected_at_upload(agpm):
    """The device path samples simple graphs (every builder — from_edges, the
    loaders' edge lists, the generators, device ingest — drops self-loops); a CSR
    handed over with a self-loop is refused loudly at upload, not sampled wrongly."""
    g = agpm.rmat(10, 8, seed=4).relabel_by_degree()
    off, nbr = g.arrays()
    lists = [list(nbr[off[u]:off[u + 1]]) for u in range(len(off) - 1)]
    lists[5] = sorted(lists[5] + [5])
    loff = np.zeros(len(lists) + 1, np.uint64)
    loff[1:] = np.cumsum([len(x) for x in lists])
    lnbr = np.array([x for li in lists for x in li], np.uint32)
    with pytest.raises(ValueError, match="self-loops"):
        agpm.DeviceGraph(begin=loff, neighbors=lnbr, edge_count=g.edge_count)
    agpm.DeviceGraph(begin=off, neighbors=nbr, edge_count=g.edge_count)  # the same graph without the loop
