"""CPU: the product's host logic (libagpm_b200.so, no GPU needed) against the reference.

Pattern/plan compiler (plan.cpp:57-137), pattern errors (pattern.cpp:77-165),
graph construction and generators (csr_graph.cpp, test_graphs.hpp), binary CSR
I/O, statistics — all through the C-ABI, compared with golden outputs of the
compiled reference.
"""
import hashlib
import json
import os
import re

import numpy as np
import pytest

from paper_2405_03488_b200._abi import Accumulator

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def h64(*arrays):
    m = hashlib.sha256()
    for a in arrays:
        m.update(np.ascontiguousarray(a).tobytes())
    return m.hexdigest()[:32]


def test_every_plan_matches_reference(agpm):
    """19 builtins x {eager, lazy} x symmetry on/off x induced overrides + custom specs,
    every field of ExecutionPlan and the scaling-rule text."""
    g = load("plans.json")
    assert len(g["plans"]) > 200
    for key, want in g["plans"].items():
        spec, mode, sym, ind = key.split("|")
        plan = agpm.compile_plan(spec, int(mode), bool(int(sym)), ind)
        assert plan.to_dict() == want["plan"], key
        assert agpm.scaling_rule_text(plan) == want["rule"], key
        assert agpm.plan_verifies_each_edge_once(plan), key


def test_pattern_errors_match_reference(agpm):
    g = load("plans.json")["errors"]
    codes = {2: agpm.PatternError, 1: ValueError}
    for key, (status, msg) in g.items():
        spec, ind = key.split("|")
        assert status in codes, key
        with pytest.raises(codes[status]) as e:
            agpm.compile_plan(spec, "eager", True, ind)
        assert str(e.value) == msg, key


def test_builtins_and_automorphisms(agpm):
    g = load("plans.json")["automorphisms"]
    assert agpm.builtin_pattern_names() == list(g.keys()) or sorted(agpm.builtin_pattern_names()) == sorted(g)
    for name, cnt in g.items():
        assert agpm.automorphism_count(name) == cnt


def test_generators_and_from_edges(agpm):
    """er_graph (test_graphs.hpp:37-43) and from_edges (csr_graph.cpp:46-72) reproduce the
    reference CSR byte for byte."""
    g = load("graphs.json")
    for key, r in g.items():
        if key.startswith("er|"):
            _, n, p, s = key.split("|")
            graph = agpm.er_graph(int(n), float(p), int(s))
        else:
            graph = agpm.CsrGraph.from_edges(np.array(r["edges"], np.uint32))
        off, nbr = graph.arrays()
        assert graph.edge_count == r["m"], key
        assert h64(off, nbr) == r["hash"], key


def test_from_edges_edge_cases(agpm):
    empty = agpm.CsrGraph.from_edges(np.zeros((0, 2), np.uint32))
    assert empty.vertex_count == 0 and empty.edge_count == 0
    loops = agpm.CsrGraph.from_edges([[2, 2], [0, 1], [1, 0]])
    assert loops.vertex_count == 3 and loops.edge_count == 1  # self-loop still counts toward n
    iso = agpm.CsrGraph.from_edges([[3, 4]], 10)
    off, nbr = iso.arrays()
    assert iso.vertex_count == 10 and off.tolist()[:4] == [0, 0, 0, 0]


def test_relabel_and_orient(agpm):
    g = agpm.rmat(10, 8, seed=5)
    r = g.relabel_by_degree()
    off, nbr = r.arrays()
    deg = np.diff(off)
    assert (np.diff(deg) >= 0).all()  # id order == (degree, id) order
    assert r.edge_count == g.edge_count and sorted(np.diff(g.arrays()[0]).tolist()) == deg.tolist()
    for u in range(r.vertex_count):
        lst = nbr[off[u]:off[u + 1]]
        assert (np.diff(lst.astype(np.int64)) > 0).all() and u not in lst
    o = r.orient_by_degree()  # on a relabelled graph: the upper suffix of every list
    ooff, onbr = o.arrays()
    assert o.oriented and len(onbr) == r.edge_count
    for u in range(0, r.vertex_count, 7):
        lst = nbr[off[u]:off[u + 1]]
        assert onbr[ooff[u]:ooff[u + 1]].tolist() == lst[lst > u].tolist()


def test_binary_io_roundtrip(agpm, tmp_path, ref):
    g = agpm.er_graph(50, 0.2, 7)
    path = str(tmp_path / "g.bin")
    g.write_binary(path)
    g2 = agpm.CsrGraph.load(path)
    a, b = g.arrays(), g2.arrays()
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and g2.edge_count == g.edge_count
    rg = ref.load(path)  # the reference's load_binary_csr reads the product's file
    ra = rg.arrays()
    assert np.array_equal(a[0], ra[0]) and np.array_equal(a[1], ra[1])
    txt = tmp_path / "g.txt"
    txt.write_text("# comment\n% also\n\n0 1\n1 2\n2 0\n")
    t = agpm.CsrGraph.load(str(txt))
    assert t.vertex_count == 3 and t.edge_count == 3
    bad = tmp_path / "bad.txt"
    bad.write_text("0 1\nnope 2\n")
    with pytest.raises(agpm.ParseError, match="line 2"):
        agpm.CsrGraph.load(str(bad))
    with pytest.raises(agpm.IoError):
        agpm.CsrGraph.load(str(tmp_path / "missing.bin"))


def test_stats_through_abi(agpm):
    g = load("stats.json")
    for q, z in g["inv_norm_cdf"]:
        assert agpm.inv_norm_cdf(q).hex() == z
    for case in g["predicted_error"]:
        rep = agpm.predicted_error(Accumulator(*case["acc"]), case["delta"])
        assert rep.mu.hex() == case["mu"] and rep.epsilon_hat.hex() == case["epsilon_hat"]
    assert abs(agpm.inv_norm_cdf(0.975) - 1.959964) < 1e-5  # test_ns_engine.cpp:17
    worst = max(abs(agpm.norm_cdf(agpm.inv_norm_cdf(q)) - q) for q in np.linspace(0.001, 0.999, 2001))
    assert worst <= 1e-10  # acceptance criterion 12
    with pytest.raises(ValueError):
        agpm.inv_norm_cdf(1.0)


def test_abi_exports_every_declared_symbol(agpm):
    """libagpm_b200.so exports every function include/agpm_b200.h declares."""
    src = open(os.path.join(ROOT, "include", "agpm_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(agpm_[a-z0-9_]+)\s*\(", src))
    assert len(names) > 35
    lib = agpm.lib()
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing


def test_device_calls_fail_loudly_without_gpu(agpm):
    """No CPU fallback: without a CUDA device, device entry points raise."""
    if agpm.device_count() > 0:
        pytest.skip("a GPU is visible")
    g = agpm.er_graph(20, 0.3, 1)
    with pytest.raises((agpm.NoDeviceError, agpm.CudaError)):
        agpm.DeviceGraph(g)
