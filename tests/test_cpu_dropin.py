"""CPU: a reference-style C++ caller compiles against include/agpm/agpm.hpp,
links libagpm_b200.so and gets the reference's answers for the host parts."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    exe = str(tmp_path / "dropin")
    lib = os.path.join(ROOT, "paper_2405_03488_b200")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "dropin_host.cpp"), "-L", lib, "-lagpm_b200",
                    f"-Wl,-rpath,{lib}", "-o", exe], check=True)
    return exe


def test_dropin_header_host_calls(agpm, tmp_path):
    out = subprocess.run([_build(tmp_path)], check=True, capture_output=True, text=True).stdout
    assert "plan 4clique k=4 steps=2 seed_ordered=1 rule='m * |S_2| * |S_3|'" in out
    assert "hand-built 4-cycle rule='m * |S_2| * |S_3|'" in out
    assert "pattern_error ok" in out
    assert "graph n=4 m=6" in out
    assert "eps_hat=1.38590" in out  # test_ns_engine.cpp:86
    assert "keep p=0.05533 colors=18" in out  # test_gs_engine.cpp:14-34
    # cost model through the header (the C entry points are reference-pinned in test_cpu_cost.py)
    assert "cone 2.200e-05..4.700e-05 gs 2.250e-08 -> GS" in out
    # K4: 4 triangles (brute force), 2 through any edge (= gamma), 12 arcs; SeedIndex.arc = the
    # reference's upper_bound(prefix) arc (ns_engine.cpp:18-23)
    assert "brute triangles=4 through(0,1)=2 gamma=2 seeds=12 arc0=(0,1) arc11=(3,2)" in out


@pytest.mark.gpu
def test_dropin_header_device_calls(agpm, tmp_path):
    out = subprocess.run([_build(tmp_path), "--device"], check=True, capture_output=True, text=True).stdout
    import re
    est = float(re.search(r"K4 4-cliques ~ ([0-9.]+)", out).group(1))
    assert abs(est - 1.0) < 0.1  # K4 holds exactly one 4-clique; eps = 5 %
    assert "converged=1" in out
    assert "exact triangles=4 4cliques=1" in out
    assert "gs c=1 estimate=4.0 raw=4" in out
    # colours {0,1,0,1} on K4 keep edges 0-2 and 1-3; merging both colours restores K4
    assert "colored same=2 merged same=6 merged triangles=4" in out
    assert re.search(r"draw value=(\S+) hit=(\d)", out).groups() == \
        re.search(r"draw with seed index value=(\S+) hit=(\d)", out).groups()
    assert "aba 0 1 0 1" in out  # no stale device mirror for a freed graph's successor
    assert "same=1" in out  # workers -> GPUs: identical result (one rank on a 1-GPU box)
