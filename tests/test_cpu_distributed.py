"""CPU, world_size 2 (gloo): the host side of the multi-GPU drivers.

On GPUs the sharded online loop (csrc/ns_device.cu online_loop) runs per rank:
agpm_ns_shard_round says which ids this rank draws in the round, the rank folds
them into 1000-sample window records, the records are all-gathered (NCCL) in
rank order and every rank runs the stop test over the gathered prefix. Here the
same loop runs on CPU ranks: the PRODUCT's partition function (the C-ABI call,
no device needed) decides the ids, the oracle stands in for the sampling kernel
only, gloo carries the records. The result must equal the single-process
reference-semantics run_ns_online (workers = 1): same stop n, windows, hits;
sums to reduction-order rounding. (The native loop itself is checked on the GPU
against the 1-rank run: tests/test_gpu_multi.py.)
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WINDOW = 1000


def window_records(values, window, nrec):
    """(n, hits, sum, squared_sum) per window of consecutive samples, padded to nrec records."""
    out = np.zeros((nrec, 4), np.float64)
    for w in range((len(values) + window - 1) // window):
        seg = values[w * window:(w + 1) * window]
        s = sq = 0.0
        for x in seg:
            s += x
            sq += x * x
        out[w] = (len(seg), np.count_nonzero(seg), s, sq)
    return out


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

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, p, sg, pat, eps, delta, seed, max_samples, per_rank = case
    g = A.er_graph(n, p, sg)
    off, nbr = g.arrays()
    plan = A.compile_plan(pat)
    O = Oracle()
    z = A.inv_norm_cdf(1.0 - delta / 2.0)
    acc = A.Accumulator()
    windows, launched, batch, stopped, rep = 0, 0, per_rank, False, None
    while launched < max_samples and not stopped:
        sr = A.shard_round(launched, batch, WINDOW, max_samples, rank, world)
        vals = np.zeros(0)
        if sr.count:
            vals, _, _ = O.draw_records(off, nbr, g.edge_count, plan, seed, sr.first_id, sr.count)
        local = torch.from_numpy(window_records(vals, WINDOW, sr.windows_per_rank))
        parts = [torch.zeros_like(local) for _ in range(world)]
        dist.all_gather(parts, local)
        recs = torch.cat(parts).numpy()[: sr.valid_windows]
        for nn, hh, s, sq in recs:  # the stop test after every window, in id order
            acc.n += int(nn)
            acc.hits += int(hh)
            acc.sum += float(s)
            acc.squared_sum += float(sq)
            windows += 1
            rep = O.predicted_error(acc, delta)
            if rep.epsilon_hat <= eps or acc.n >= max_samples:
                stopped = True
                break
        launched += sr.round_ids
        batch = min(batch * 2, 16 * per_rank)
    assert z > 0
    out_q.put((rank, acc.n, acc.hits, acc.sum, acc.squared_sum, windows, rep.epsilon_hat <= eps, rep.epsilon_hat))
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

    total = all_reduce_sum(O.exact_count_shard(off, nbr, g.edge_count, plan, rank, world))
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


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_round_partitions_ids(agpm, world):
    """agpm_ns_shard_round (the online loop's id partition): the ranks' blocks
    tile the round's ids in rank order, every block starts on a window boundary,
    the valid window records are exactly the gathered prefix, and the cap cuts
    the round without gaps."""
    for window, batch, max_samples in ((1000, 4000, 10**9), (1000, 2000, 9500), (10, 30, 125), (7, 7, 50)):
        launched = 0
        while launched < max_samples:
            rs = [agpm.shard_round(launched, batch, window, max_samples, r, world) for r in range(world)]
            rnd = rs[0].round_ids
            assert rnd == min(world * batch, max_samples - launched)
            nxt = launched
            recs = 0
            for r, sr in enumerate(rs):
                assert sr.round_ids == rnd and sr.windows_per_rank == batch // window
                if sr.count:
                    assert sr.first_id == nxt and sr.first_id % window == launched % window
                    assert recs == r * sr.windows_per_rank  # earlier ranks were full
                    recs += (sr.count + window - 1) // window
                nxt += sr.count
            assert nxt == launched + rnd and recs == rs[0].valid_windows
            launched += rnd
            if launched > 10 * world * batch:
                break
    with pytest.raises(ValueError):
        agpm.shard_round(0, 1500, 1000, 10**9, 0, 2)  # batch not a window multiple
