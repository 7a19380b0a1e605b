"""GPU: BASELINE.json configs at their full sizes.

config 1  triangle, er_graph(10^4, 20/9999, 1) relabelled: 2^20 samples seed 1
          (fixed budget) and the exact count, against the oracle.
config 2  4-clique, RMAT-20 ef16 relabelled, run_ns_online to 1 %@95 %: the device
          run stops at the same n with the same hits as the oracle's own online run
          (the C restatement, ~0.5 M samples), and the estimate is within the bound
          of the exact count.
config 4  needle: ER n = 2^22, avg degree 8, 1000 planted 5-cliques — the
          region split finds every planted clique exactly.
config 4  the colour-GS dense leg: with tau = 10 about a third of the planted
          K5s lie entirely in the dense region, so c = 4 colourings repeated to
          1 %@95 % estimate a real count there, checked against the exact count.
(configs 3 / 5 at size: tests/test_gpu_scale.py.)
"""
import pytest

pytestmark = pytest.mark.gpu


def test_config1(agpm, oracle):
    g = agpm.er_graph(10000, 20 / 9999, 1).relabel_by_degree()
    off, nbr = g.arrays()
    plan = agpm.compile_plan("triangle")
    dg = agpm.DeviceGraph(g)
    exact = agpm.exact_count(dg, plan)
    assert exact == oracle.exact_count(off, nbr, g.edge_count, plan) == 1380  # SURVEY §6 probe
    acc = agpm.run_fixed_budget(dg, plan, 1 << 20, 1)
    o = oracle.fixed_budget(off, nbr, g.edge_count, plan, 1 << 20, 1)
    assert acc.n == o.n == 1 << 20 and acc.hits == o.hits
    assert abs(acc.sum - o.sum) <= 1e-12 * o.sum
    assert abs(acc.sum / acc.n - exact) < 0.05 * exact


@pytest.mark.slow
def test_config2_online_parity(agpm, oracle):
    g = agpm.rmat(20, 16, 0.57, 0.19, 0.19, seed=1).relabel_by_degree()
    off, nbr = g.arrays()
    plan = agpm.compile_plan("4clique")
    dg = agpm.DeviceGraph(g)
    r = agpm.run_ns_online(dg, plan, 0.01, 0.05, agpm.OnlinePolicy(), seed=1)
    o = oracle.ns_online(off, nbr, g.edge_count, plan, 0.01, 0.05, agpm.OnlinePolicy(), 1)
    assert r.report.converged and o.report.converged
    assert r.report.n == o.report.n and r.windows == o.windows and r.accumulator.hits == o.accumulator.hits
    assert abs(r.report.mu - o.report.mu) <= 1e-12 * o.report.mu
    # the exact 4-clique count on the oriented DAG (device) and the 1 %@95 % promise
    exact = agpm.exact_count(agpm.DeviceGraph(g.orient_by_degree()), plan)
    assert abs(r.report.mu - exact) <= 0.02 * exact


@pytest.mark.slow
def test_config4_needle(agpm):
    n = 1 << 22
    g = agpm.er_fast(n, n * 4, seed=4, planted_k=5, planted_count=1000).relabel_by_degree()
    dg = agpm.DeviceGraph(g)
    plan = agpm.compile_plan("5clique")
    exact = agpm.exact_count(dg, plan)
    assert exact >= 1000
    res = agpm.region_split(dg, plan, 16, dense="gs", colors=4, repeats=8)
    assert res.c_sparse + (int(res.c_dense) if res.dense_exact else 0) <= exact
    full = agpm.region_split(dg, plan, 16, dense="exact")
    assert full.estimate == exact


@pytest.mark.slow
def test_config4_gs_dense_leg(agpm):
    """Config 4's c = 4 colour-GS leg on a dense region that holds planted K5s
    (gs_engine.cpp:42-75 per colouring, the online detector over colourings):
    sparse part exact, dense part within the error bound of the exact count."""
    n = 1 << 22
    g = agpm.er_fast(n, n * 4, seed=4, planted_k=5, planted_count=1000).relabel_by_degree()
    dg = agpm.DeviceGraph(g)
    plan = agpm.compile_plan("5clique")
    exact = agpm.exact_count(dg, plan)
    tau = 10  # planted vertices have degree ~ Poisson(8) + 4: many reach the dense region
    ex = agpm.region_split(dg, plan, tau, dense="exact")
    assert ex.estimate == exact
    dense_truth = exact - ex.c_sparse
    assert dense_truth >= 100  # a real population of K5s for GS to estimate
    gs = agpm.region_split(dg, plan, tau, dense="gs", colors=4, eps=0.01, delta=0.05, repeats=200000, seed=11)
    assert gs.c_sparse == ex.c_sparse
    assert gs.dense_ns.report.converged and gs.dense_epsilon_hat <= 0.01
    # 1 %@95 %: allow 3 eps (a ~1-in-10^3 event) so the test is not flaky
    assert abs(gs.c_dense - dense_truth) <= 0.03 * dense_truth, (gs.c_dense, dense_truth, gs.dense_ns.windows)
