"""GPU: the native multi-rank drivers against the 1-rank run.

The sharded online loop (agpm_ns_online_sharded), the sharded fixed budget and
the sharded exact count run with `world` ranks of a local communicator group —
one host thread per rank; on this one-GPU box the ranks share the device, each
with its own stream and scratch, exchanging window records by stream-ordered
peer copies behind a host barrier (no kernel waits on another rank) — and with
a 1-rank NCCL communicator (the torchrun path's transport). Every rank must
reproduce the single-GPU result: stop n, windows, hits and the window-fold sums
bit for bit (the gathered records are the single-GPU records in the same
order), fixed-budget n and hits exactly, exact counts exactly.
"""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run_ranks(agpm, world, body):
    group = agpm.LocalGroup(world)
    out, errs = [None] * world, []

    def run(r):
        try:
            agpm.lib().agpm_set_device(0)
            comm = group.comm(r)
            try:
                out[r] = body(comm, r)
            finally:
                comm.close()
        except Exception as e:  # surfaced below
            errs.append(e)

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not errs, errs
    return out


@pytest.fixture(scope="module")
def rmat16(agpm):
    return agpm.rmat(16, 16, seed=1).relabel_by_degree()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("spec,eps,max_samples", [("4clique", 0.01, 10**9), ("4cycle", 0.005, 10**9),
                                                  ("triangle", 1e-4, 123_456)])  # the last hits the cap
def test_online_sharded_equals_single(agpm, rmat16, world, spec, eps, max_samples):
    plan = agpm.compile_plan(spec)
    pol = agpm.OnlinePolicy(max_samples=max_samples)
    dg = agpm.DeviceGraph(rmat16)
    single = agpm.run_ns_online(dg, plan, eps, 0.05, pol, seed=7)

    def body(comm, r):
        mine = agpm.DeviceGraph(rmat16)  # each rank its own replica
        return agpm.run_ns_online_sharded(comm, mine, plan, eps, 0.05, pol, seed=7)

    for res in _run_ranks(agpm, world, body):
        assert (res.report.n, res.windows, res.accumulator.hits) == (single.report.n, single.windows,
                                                                     single.accumulator.hits)
        assert res.accumulator.sum.hex() == single.accumulator.sum.hex()
        assert res.accumulator.squared_sum.hex() == single.accumulator.squared_sum.hex()
        assert res.report.epsilon_hat.hex() == single.report.epsilon_hat.hex()
        assert bool(res.report.converged) == bool(single.report.converged)
    if max_samples < 10**9:
        assert single.report.n == max_samples and not single.report.converged


@pytest.mark.parametrize("world", [2, 4])
def test_fixed_budget_and_exact_sharded(agpm, rmat16, world):
    plan = agpm.compile_plan("4clique")
    dg = agpm.DeviceGraph(rmat16)
    single = agpm.run_fixed_budget(dg, plan, 1_000_003, 5)
    exact = agpm.exact_count(agpm.DeviceGraph(rmat16.orient_by_degree()), plan)

    def body(comm, r):
        acc = agpm.run_fixed_budget_sharded(comm, agpm.DeviceGraph(rmat16), plan, 1_000_003, 5)
        cnt = agpm.exact_count_sharded(comm, agpm.DeviceGraph(rmat16.orient_by_degree()), plan)
        return acc, cnt

    for acc, cnt in _run_ranks(agpm, world, body):
        assert (acc.n, acc.hits) == (single.n, single.hits)
        assert abs(acc.sum - single.sum) <= 1e-12 * single.sum
        assert cnt == exact


def test_nccl_single_rank(agpm, rmat16):
    """The NCCL transport (one process per GPU under torchrun) with one rank:
    communicator setup, the all-gather in the online loop, the exact-count exchange."""
    agpm.lib().agpm_set_device(0)
    comm = agpm.Comm.nccl(0, 1, agpm.nccl_unique_id())
    assert comm.info() == {"rank": 0, "world": 1, "device": 0, "nccl": True}
    plan = agpm.compile_plan("4clique")
    dg = agpm.DeviceGraph(rmat16)
    single = agpm.run_ns_online(dg, plan, 0.01, 0.05, agpm.OnlinePolicy(), seed=3)
    res = agpm.run_ns_online_sharded(comm, dg, plan, 0.01, 0.05, agpm.OnlinePolicy(), seed=3)
    assert (res.report.n, res.accumulator.hits) == (single.report.n, single.accumulator.hits)
    assert res.accumulator.sum.hex() == single.accumulator.sum.hex()
    o = agpm.DeviceGraph(rmat16.orient_by_degree())
    assert agpm.exact_count_sharded(comm, o, plan) == agpm.exact_count(o, plan)
    comm.close()


def test_threads_share_one_view(agpm, rmat16):
    """Several host threads sampling ONE view concurrently (the lazy dense-core /
    twin-arc index builds are locked and published only when built; each thread
    has its own stream and scratch): every thread gets the single-thread records."""
    plan = agpm.compile_plan("4clique")
    dg = agpm.DeviceGraph(rmat16)
    want = agpm.draw_samples(agpm.DeviceGraph(rmat16), plan, 1, 0, 1 << 18)
    got, errs = [None] * 4, []

    def run(i):
        try:
            agpm.lib().agpm_set_device(0)
            got[i] = agpm.draw_samples(dg, plan, 1, 0, 1 << 18)
        except Exception as e:
            errs.append(e)

    ts = [threading.Thread(target=run, args=(i,)) for i in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    assert not errs, errs
    for v, h, b in got:
        assert np.array_equal(v.view(np.uint64), want[0].view(np.uint64)) and np.array_equal(b, want[2])
