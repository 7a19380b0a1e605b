"""CPU, world_size 2 (gloo): the sharded online driver of paper_2405_03488_b200.distributed.

Each rank draws its shard of global sample ids (here with the C oracle as the
per-rank sampler — on GPUs the sampling kernel), reduces them to window
moments, the ranks all-gather the moments and replay the window loop. The
result must equal the single-process reference-semantics run_ns_online
(workers = 1): same stop n, windows, hits; sums to reduction-order rounding.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, out_q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch

    import paper_2405_03488_b200 as A
    from oracle_bindings import Oracle
    from paper_2405_03488_b200 import distributed as D

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, p, sg, pat, eps, delta, seed, max_samples, per_rank = case
    g = A.er_graph(n, p, sg)
    off, nbr = g.arrays()
    plan = A.compile_plan(pat)
    O = Oracle()

    def sample_moments(first, count):
        v, h, b = O.draw_records(off, nbr, g.edge_count, plan, seed, first, count)
        return D.window_moments(v, 1000)

    def all_gather(local):
        t = torch.from_numpy(local)
        parts = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        return torch.cat(parts).numpy()

    m = D.run_ns_online_sharded(sample_moments, all_gather, rank, world, eps, delta, window=1000,
                                max_samples=max_samples, per_rank=per_rank)
    out_q.put((rank, m.acc.n, m.acc.hits, m.acc.sum, m.acc.squared_sum, m.windows, m.report.converged,
               m.report.epsilon_hat))
    dist.destroy_process_group()


@pytest.mark.parametrize("case", [
    (200, 0.08, 71, "4clique", 0.2, 0.05, 31, 10**9, 4000),
    (100, 0.1, 66, "triangle", 0.05, 0.05, 3, 10**9, 3000),
    (60, 0.2, 17, "4cycle", 0.01, 0.05, 5, 9500, 2000),  # hits the (non-window-aligned) cap
])
def test_sharded_online_equals_single_process(agpm, oracle, case):
    n, p, sg, pat, eps, delta, seed, max_samples, per_rank = case
    g = agpm.er_graph(n, p, sg)
    off, nbr = g.arrays()
    pol = agpm.OnlinePolicy(max_samples=max_samples)
    ref = oracle.ns_online(off, nbr, g.edge_count, agpm.compile_plan(pat), eps, delta, pol, seed)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for _, nn, hits, s, sq, windows, conv, eh in res:
        assert nn == ref.report.n and hits == ref.accumulator.hits and windows == ref.windows
        assert bool(conv) == bool(ref.report.converged)
        assert abs(s - ref.accumulator.sum) <= 1e-12 * max(1.0, abs(ref.accumulator.sum))
        assert abs(sq - ref.accumulator.squared_sum) <= 1e-12 * max(1.0, abs(ref.accumulator.squared_sum))
    assert res[0][1:] == res[1][1:]  # every rank reaches the same decision


def _exact_worker(rank, world, port, case, out_q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch

    import paper_2405_03488_b200 as A
    from oracle_bindings import Oracle
    from paper_2405_03488_b200 import distributed as D

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, p, sg, pat = case
    g = A.er_graph(n, p, sg).relabel_by_degree()
    off, nbr = g.arrays()
    plan = A.compile_plan(pat)
    O = Oracle()

    def all_reduce_sum(x):
        t = torch.tensor([x], dtype=torch.int64)
        dist.all_reduce(t)
        return int(t.item())

    total = D.exact_count_sharded(lambda r, w: O.exact_count_shard(off, nbr, g.edge_count, plan, r, w),
                                  all_reduce_sum, rank, world)
    out_q.put((rank, total))
    dist.destroy_process_group()


@pytest.mark.parametrize("case", [(200, 0.08, 71, "4clique"), (150, 0.1, 5, "4cycle"), (120, 0.15, 9, "house")])
def test_sharded_exact_count_equals_single_process(agpm, oracle, case):
    """Sharded exact counting (interleaved 32-arc chunks per rank, u64 partials
    all-reduced) gives the single-process exact_count on every rank."""
    n, p, sg, pat = case
    g = agpm.er_graph(n, p, sg).relabel_by_degree()
    off, nbr = g.arrays()
    want = oracle.exact_count(off, nbr, g.edge_count, agpm.compile_plan(pat))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exact_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert all(t == want for _, t in res)


@pytest.mark.parametrize("nshards", [1, 2, 5])
def test_oracle_shards_sum_to_exact_count(agpm, oracle, nshards):
    g = agpm.rmat(9, 8, seed=2).relabel_by_degree()
    off, nbr = g.arrays()
    for pat in ("triangle", "4clique", "4cycle"):
        plan = agpm.compile_plan(pat)
        parts = [oracle.exact_count_shard(off, nbr, g.edge_count, plan, r, nshards) for r in range(nshards)]
        assert sum(parts) == oracle.exact_count(off, nbr, g.edge_count, plan)
