"""GPU parity at the big configs' own scale (BASELINE.json configs 3 and 5).

The samplers that only run on big graphs — the frontier phases (plans that are not
core suffixes; any plan above 2^26 vertices), hub-list
(long-driver) paths, the partial dense core, the twin-arc hints (built by
prepare() here; lazily only after `arcs` sampled ids) — are pinned here against the oracle on the
graphs themselves, not on scaled-down stand-ins:

* config 3: RMAT-22 ef16 relabelled, 4-cycle on the flat (auto: the fast class
  with bound list owners inside [lo, hi)), frontier and warp samplers, 4-clique on
  flat and frontier, the house (auto = frontier);
* config 5 class: RMAT-25 ef16 relabelled, 4-clique on the flat (auto) and the
  frontier samplers, and RMAT-27 itself (auto = frontier) when the host can hold
  the oracle's copy of the 4.2 B-arc CSR.

Each graph is built on the device (== the host builders, tests/test_gpu_ingest.py)
and downloaded for the oracle, so both sides read the same arrays. Per-sample
records (value bits, hit, bindings) are compared at three id offsets (0, 2^30,
2^40), and run_ns_online(1 %, 5 %) must stop at the oracle's n with its hits and
sums (ns_engine.cpp:27-53, 106-140). The oracle runs its multi-threaded
variants (orc_draw_records_mt / orc_ns_online_mt: same streams, in-order
accumulation — bit-identical to the sequential functions, test_cpu_oracle.py).
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

OFFSETS = (0, 1 << 30, 1 << 40)
COUNT = 1 << 18  # >= 2^18: the batch size where the auto strategy leaves the warp sampler
STRATEGY = {"auto": 0, "warp": 1, "lane": 2, "frontier": 3, "flat": 5}


def _graph(agpm, scale):
    dg = agpm.rmat_device(scale, 16, 0.57, 0.19, 0.19, seed=1, relabel=True)
    b, e, nb = dg.download()
    return dg, (b, e, nb), dg.info()


def _records_equal(agpm, oracle, dg, host, m, plan, first, count):
    b, e, nb = host
    v, h, bd = agpm.draw_samples(dg, plan, 1, first, count)
    ov, oh, ob = oracle.draw_records_mt(b, nb, m, plan, 1, first, count, end=e)
    bad = np.flatnonzero((v.view(np.uint64) != ov.view(np.uint64)) | (h != oh) | (bd != ob).any(axis=1))
    assert bad.size == 0, (f"{bad.size} of {count} records differ from the oracle at id offset {first}; "
                           f"first id {first + int(bad[0])}: device {v[bad[0]]!r} {bd[bad[0]].tolist()} "
                           f"oracle {ov[bad[0]]!r} {ob[bad[0]].tolist()}")
    return int(h.sum())


def _online_equal(agpm, oracle, dg, host, m, plan):
    b, e, nb = host
    pol = agpm.OnlinePolicy()
    r = agpm.run_ns_online(dg, plan, 0.01, 0.05, pol, seed=1)
    o = oracle.ns_online_mt(b, nb, m, plan, 0.01, 0.05, pol, 1, end=e)
    assert r.report.converged and o.report.converged
    assert (r.report.n, r.windows, r.accumulator.hits) == (o.report.n, o.windows, o.accumulator.hits)
    assert abs(r.accumulator.sum - o.accumulator.sum) <= 1e-12 * o.accumulator.sum
    assert abs(r.accumulator.squared_sum - o.accumulator.squared_sum) <= 1e-12 * o.accumulator.squared_sum
    return r


@pytest.fixture(scope="module")
def rmat22(agpm):
    return _graph(agpm, 22)


@pytest.mark.parametrize("spec,strategy", [("4cycle", "auto"), ("4cycle", "frontier"), ("4clique", "auto"),
                                           ("4clique", "frontier"), ("4cycle", "warp"), ("triangle", "auto"),
                                           ("house", "auto")])
def test_config3_records(agpm, oracle, rmat22, spec, strategy):
    dg, host, info = rmat22
    plan = agpm.compile_plan(spec)
    agpm.set_strategy(strategy)
    try:
        if strategy == "auto":  # core-suffix plans (cliques, the 4-cycle) run flat, the rest on the frontier phases
            assert agpm.strategy_for(dg, plan, COUNT) == ("frontier" if spec == "house" else "flat")
        hits = [_records_equal(agpm, oracle, dg, host, info["edge_count"], plan, f, COUNT) for f in OFFSETS]
    finally:
        agpm.set_strategy("auto")
    assert sum(hits) > 0


@pytest.mark.parametrize("spec,strategy", [("4cycle", "auto"), ("4cycle", "frontier"), ("4clique", "auto"),
                                           ("4clique", "frontier")])
def test_config3_records_with_twin_hints(agpm, oracle, rmat22, spec, strategy):
    """The same records once the view's twin-arc index exists (built lazily only
    after `arcs` sampled ids; prepare() builds it now): hinted seed ranges at scale."""
    dg, host, info = rmat22
    before = dg.info()["device_bytes"]
    dg.prepare()
    assert dg.info()["device_bytes"] >= before  # grows by 4 B per arc on the first call
    plan = agpm.compile_plan(spec)
    agpm.set_strategy(strategy)
    try:
        _records_equal(agpm, oracle, dg, host, info["edge_count"], plan, OFFSETS[1], COUNT)
    finally:
        agpm.set_strategy("auto")


@pytest.mark.parametrize("spec", ["4clique", "5clique"])
def test_config3_sorted_launch(agpm, oracle, rmat22, spec):
    """A launch of 2^20 ids: the flat sampler works through it in seed-sorted order (arc
    key for the 4-clique, composite key for the 5-clique) with shared first steps
    (ns_flat.cu: flat_order) — same records as the oracle at scale."""
    dg, host, info = rmat22
    plan = agpm.compile_plan(spec)
    assert agpm.strategy_for(dg, plan, 1 << 20) == "flat"
    assert _records_equal(agpm, oracle, dg, host, info["edge_count"], plan, OFFSETS[1] + 7, 1 << 20) > 0


def test_config3_online(agpm, oracle, rmat22):
    dg, host, info = rmat22
    r = _online_equal(agpm, oracle, dg, host, info["edge_count"], agpm.compile_plan("4cycle"))
    assert r.report.n >= 1000


@pytest.fixture(scope="module")
def rmat25(agpm):
    return _graph(agpm, 25)


@pytest.mark.parametrize("spec,strategy", [("4clique", "auto"), ("4clique", "frontier"), ("4cycle", "auto")])
def test_config5_class_records(agpm, oracle, rmat25, spec, strategy):
    dg, host, info = rmat25
    assert info["vertex_count"] == 1 << 25  # 256 K core; the auto strategy sends core-suffix plans to flat up to 2^26
    plan = agpm.compile_plan(spec)
    agpm.set_strategy(strategy)
    try:
        hits = [_records_equal(agpm, oracle, dg, host, info["edge_count"], plan, f, COUNT) for f in OFFSETS]
    finally:
        agpm.set_strategy("auto")
    assert sum(hits) > 0


@pytest.mark.parametrize("spec", ["4clique", "5clique"])
def test_config5_class_sorted_launch(agpm, oracle, rmat25, spec):
    """RMAT-25, one 2^20-id launch: seed-sorted order on the arc key (every plan above 2^22 vertices)."""
    dg, host, info = rmat25
    _records_equal(agpm, oracle, dg, host, info["edge_count"], agpm.compile_plan(spec), OFFSETS[0] + 3, 1 << 20)


def test_config5_class_online(agpm, oracle, rmat25):
    dg, host, info = rmat25
    dg.prepare()  # twin-arc hints on: the online run and the records after it use them
    _records_equal(agpm, oracle, dg, host, info["edge_count"], agpm.compile_plan("4clique"), OFFSETS[2], COUNT)
    _online_equal(agpm, oracle, dg, host, info["edge_count"], agpm.compile_plan("4clique"))


def _host_bytes():
    try:
        import psutil

        return psutil.virtual_memory().available
    except Exception:
        return 0


@pytest.mark.skipif(_host_bytes() < (48 << 30), reason="host RAM cannot hold the oracle's RMAT-27 copy")
def test_config5_rmat27(agpm, oracle):
    """Config 5 itself: RMAT-27 ef16 (2.1 B edges, int64 offsets), 4-clique —
    records at three offsets and the 1 %@95 % online stop n vs the oracle."""
    dg, host, info = _graph(agpm, 27)
    assert info["arcs"] > (1 << 31)  # arc offsets beyond int32 (u64 offsets, csr_graph.hpp:26-28)
    plan = agpm.compile_plan("4clique")
    m = info["edge_count"]
    for f in OFFSETS:
        _records_equal(agpm, oracle, dg, host, m, plan, f, 1 << 16)
    _online_equal(agpm, oracle, dg, host, m, plan)
