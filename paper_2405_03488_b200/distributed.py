"""Multi-rank neighbour sampling: samples sharded by global id, moments exchanged.

SURVEY §8(e): the CSR is replicated on every GPU; global sample id i always
uses CounterRng(seed, 0, i), so an N-rank run draws exactly the samples of the
1-rank run (and of the reference with workers = 1). Per batch b, rank r draws
ids [(b*N + r)*B, (b*N + r + 1)*B) with B a multiple of the convergence window;
each rank reduces its samples to per-window moments (n, hits, sum, squared
sum), the ranks all-gather those 32-byte records (NCCL over NVLink on GPUs,
gloo in the CPU tests) — rank order is global id order — and every rank replays
the reference's window loop (ns_engine.cpp:121-137) on the gathered records,
stopping at the first window with eps_hat <= eps. Only moments cross ranks.
"""
import math

import numpy as np

from ._abi import Accumulator, Report

__all__ = ["predicted_error_py", "WindowMerger", "batch_first_id", "run_ns_online_sharded", "exact_count_sharded"]


def _inv_norm_cdf(q):
    # stats.cpp:14-55: Acklam + two Newton steps (identical operation order)
    a = [-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02, 1.383577518672690e+02,
         -3.066479806614716e+01, 2.506628277459239e+00]
    b = [-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02, 6.680131188771972e+01,
         -1.328068155288572e+01]
    c = [-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00, -2.549732539343734e+00,
         4.374664141464968e+00, 2.938163982698783e+00]
    d = [7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00, 3.754408661907416e+00]
    if not (0.0 < q < 1.0):
        raise ValueError("quantile must be inside (0,1)")
    if q < 0.02425:
        r = math.sqrt(-2.0 * math.log(q))
        z = (((((c[0] * r + c[1]) * r + c[2]) * r + c[3]) * r + c[4]) * r + c[5]) / \
            ((((d[0] * r + d[1]) * r + d[2]) * r + d[3]) * r + 1.0)
    elif q > 1.0 - 0.02425:
        r = math.sqrt(-2.0 * math.log(1.0 - q))
        z = -(((((c[0] * r + c[1]) * r + c[2]) * r + c[3]) * r + c[4]) * r + c[5]) / \
            ((((d[0] * r + d[1]) * r + d[2]) * r + d[3]) * r + 1.0)
    else:
        r = q - 0.5
        t = r * r
        z = (((((a[0] * t + a[1]) * t + a[2]) * t + a[3]) * t + a[4]) * t + a[5]) * r / \
            (((((b[0] * t + b[1]) * t + b[2]) * t + b[3]) * t + b[4]) * t + 1.0)
    for _ in range(2):
        err = 0.5 * math.erfc(-z / math.sqrt(2.0)) - q
        pdf = math.exp(-0.5 * z * z) / math.sqrt(2.0 * math.pi)
        if pdf <= 0.0:
            break
        z -= err / pdf
    return z


def predicted_error_py(n, hits, s, sq, z):
    """stats.cpp:57-70 for an accumulator (n, hits, sum, squared_sum), z = Phi^-1(1 - delta/2)."""
    rep = Report()
    rep.n = n
    rep.epsilon_hat = math.inf
    if n == 0:
        return rep
    rep.hit_rate = hits / n
    rep.mu = s / n
    if not (s > 0.0) or n < 2:
        return rep
    var = sq / n - rep.mu * rep.mu
    if var < 0.0:
        var = 0.0
    rep.sigma = math.sqrt(var / n)
    rep.epsilon_hat = z * rep.sigma / rep.mu
    return rep


def window_moments(values, window):
    """Per-window (n, hits, sum, squared_sum) of consecutive samples (host restatement of
    the device window kernel; sums are sequential here, pairwise-tree on the device)."""
    v = np.asarray(values, dtype=np.float64)
    nw = (len(v) + window - 1) // window
    out = np.zeros((nw, 4), np.float64)
    for w in range(nw):
        seg = v[w * window:(w + 1) * window]
        s = sq = 0.0
        for x in seg:
            s += x
            sq += x * x
        out[w] = (len(seg), np.count_nonzero(seg), s, sq)
    return out


class WindowMerger:
    """Replays run_ns_online's window loop on gathered window moments."""

    def __init__(self, eps, delta, max_samples):
        if not (0.0 < eps < 1.0):
            raise ValueError("error bound must be inside (0,1)")
        if not (0.0 < delta < 1.0):
            raise ValueError("delta must be inside (0,1)")
        self.eps, self.max_samples = eps, max_samples
        self.z = _inv_norm_cdf(1.0 - delta / 2.0)
        self.acc = Accumulator()
        self.windows = 0
        self.report = predicted_error_py(0, 0, 0.0, 0.0, self.z)
        self.stopped = False

    def feed(self, moments):
        """moments: [nwin, 4] (n, hits, sum, squared_sum) in global window order."""
        for n, hits, s, sq in moments:
            if self.stopped:
                break
            if n == 0:  # padding of a rank past the cap
                continue
            self.acc.n += int(n)
            self.acc.hits += int(hits)
            self.acc.sum += float(s)
            self.acc.squared_sum += float(sq)
            self.windows += 1
            self.report = predicted_error_py(self.acc.n, self.acc.hits, self.acc.sum, self.acc.squared_sum, self.z)
            if self.report.epsilon_hat <= self.eps:
                self.report.converged = 1
                self.stopped = True
            elif self.acc.n >= self.max_samples:
                self.stopped = True
        return self.stopped


def batch_first_id(batch, rank, world, per_rank):
    return (batch * world + rank) * per_rank


def run_ns_online_sharded(sample_moments, all_gather, rank, world, eps, delta, window=1000,
                          max_samples=1000000000, per_rank=None):
    """Drive a sharded run_ns_online.

    sample_moments(first_id, count) -> [ceil(count/window), 4] float64 window moments of this rank's ids;
    all_gather(local [nw, 4]) -> [world * nw, 4] in rank order.
    Returns the WindowMerger (identical on every rank)."""
    if per_rank is None:
        per_rank = 64 * window
    per_rank = max(window, (per_rank // window) * window)
    merger = WindowMerger(eps, delta, max_samples)
    nw = per_rank // window
    batch = 0
    while not merger.stopped:
        first = batch_first_id(batch, rank, world, per_rank)
        count = int(min(per_rank, max(0, max_samples - first)))
        local = np.zeros((nw, 4), np.float64)
        if count:
            m = sample_moments(first, count)  # window boundaries are global: first % window == 0
            local[: len(m)] = m
        merger.feed(all_gather(local))
        batch += 1
    return merger


def exact_count_sharded(count_shard, all_reduce_sum, rank, world):
    """Multi-rank exact_count: every rank holds the whole graph,
    counts the seeds of its interleaved 32-arc chunks (count_shard(rank, world),
    e.g. agpm.exact_count_shard on its own GPU) and the u64 partials are summed
    across ranks (NCCL all-reduce on GPUs, gloo in the CPU tests). Returns the
    total on every rank; it equals the single-GPU exact_count exactly."""
    if not (0 <= rank < world):
        raise ValueError("rank must be in [0, world)")
    return int(all_reduce_sum(int(count_shard(rank, world))))
