// Eager-verify neighbour sampling on sm_100a.
//
// One sample per lane, 32 samples per warp, persistent warps pulling 32-id
// batches from a global cursor. Per plan step every lane computes the
// bound-restricted ranges of its in-lists (lower_bound(lo), lower_bound(hi)
// from the order constraints of walker.hpp:64-69, narrowed by per-position
// hints: the precomputed upper-suffix start vtx.up and the seed arc index),
// then picks the cheapest of three exact paths:
//   single list  : |S| = |range| - #bound vertices inside it, r-th pick by
//                  index arithmetic (no scan);
//   short driver : the lane scans <= 64 driver elements itself, galloping in
//                  the other lists, hit set kept as a 64-bit mask;
//   long driver  : the whole warp intersects for that lane — 32 driver
//                  elements per chunk, one binary search per lane per other
//                  list, hit ballots staged in shared memory so the r-th
//                  candidate is found without a second intersection pass.
// All three enumerate S = (∩ in-lists) \ (∪ out-lists) \ bound, ascending,
// exactly the candidate vector of build_step_candidates (walker.hpp:30-83),
// and draw cand[next_below(|S|)] from the lane's CounterRng(seed, 0, id), so
// per-sample (value, hit, bindings) are bit-identical to draw_sample
// (ns_engine.cpp:27-53) with workers = 1.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <vector>

#include "device.cuh"
#include "rng.cuh"
#include "stats.hpp"

namespace agpm_b200 {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kSmallDriver = 64;   // lane-private scan up to this many driver elements
constexpr int kBallotWords = 64;   // shared ballots cover drivers up to 2048 elements

struct DevPlan {
  int k;
  int n_steps;
  int seed_ordered;
  int pad;
  double alpha0;  // seed_scale (plan.hpp:50-53): m or 2m
  unsigned short in_mask[AGPM_MAX_K - 2];
  unsigned short out_mask[AGPM_MAX_K - 2];
  unsigned short gt_mask[AGPM_MAX_K - 2];
  unsigned short lt_mask[AGPM_MAX_K - 2];
};

struct GraphArgs {
  const VtxInfo* __restrict__ vtx;
  const uint32_t* __restrict__ nbr;
  const unsigned long long* __restrict__ seed_arcs;
  unsigned long long arcs;
  int plain;
};

__device__ __forceinline__ uint32_t ldn(const uint32_t* p, unsigned long long i) { return __ldg(p + i); }

// first index in [lo, hi) with nbr[i] >= x (hi if none)
__device__ __forceinline__ unsigned long long lower_bound_dev(const uint32_t* nbr, unsigned long long lo,
                                                              unsigned long long hi, uint32_t x) {
  while (lo < hi) {
    unsigned long long mid = (lo + hi) >> 1;
    if (ldn(nbr, mid) < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// galloping lower_bound from a monotone cursor
__device__ __forceinline__ unsigned long long gallop_dev(const uint32_t* nbr, unsigned long long c,
                                                         unsigned long long e, uint32_t x) {
  if (c >= e || ldn(nbr, c) >= x) return c;
  unsigned long long lo = c, step = 1, hi = c + 1;
  while (hi < e && ldn(nbr, hi) < x) {
    lo = hi;
    step <<= 1;
    hi = lo + step;
  }
  if (hi > e) hi = e;
  return lower_bound_dev(nbr, lo + 1, hi, x);
}

__device__ __forceinline__ unsigned long long sectors(unsigned long long a, unsigned long long b) {
  return b > a ? ((b * 4 - 1) >> 5) - ((a * 4) >> 5) + 1 : 0;
}

// index of the (r+1)-th set bit of a 64-bit mask
__device__ __forceinline__ int nth_bit64(unsigned long long m, int r) {
  unsigned lo = (unsigned)m, hi = (unsigned)(m >> 32);
  int plo = __popc(lo);
  if (r < plo) return (int)__fns(lo, 0, r + 1);
  return 32 + (int)__fns(hi, 0, r - plo + 1);
}

template <int K, bool COUNT_BYTES>
__global__ void __launch_bounds__(kThreads) ns_sample_kernel(
    const GraphArgs g, const DevPlan p, const unsigned long long seed, const unsigned long long first_id,
    const unsigned long long count, double* __restrict__ values, uint32_t* __restrict__ bindings,
    unsigned long long* __restrict__ cursor, unsigned long long* __restrict__ bytes_out) {
  __shared__ uint32_t s_ballot[kWarps][kBallotWords];
  const int lane = threadIdx.x & 31;
  uint32_t* ballots = s_ballot[threadIdx.x >> 5];
  const uint32_t* __restrict__ nbr = g.nbr;
  unsigned long long bytes_acc = 0;

  for (;;) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(cursor, 32ull);
    base = __shfl_sync(FULL, base, 0);
    if (base >= count) break;
    const unsigned long long idx = base + lane;
    bool alive = idx < count;
    CounterRng rng(seed, 0, first_id + idx);

    // per-position state; all indexing below is static (unrolled over K)
    uint32_t bnd[K];
    unsigned long long pb[K], pe[K];      // list bounds [pb, pe)
    unsigned long long ha[K], hb[K];      // hint indices: lower_bound(hal/hbl)
    uint32_t hal[K], hbl[K];
#pragma unroll
    for (int q = 0; q < K; ++q) {
      bnd[q] = 0xffffffffu;
      pb[q] = pe[q] = ha[q] = hb[q] = 0;
      hal[q] = hbl[q] = 0;
    }
    double alpha = p.alpha0;
    int nbound = 0;
    unsigned used_mask = 0;  // positions whose offsets were read (B_min model)

    auto bind = [&](int q, uint32_t v) {
#pragma unroll
      for (int t = 0; t < K; ++t)
        if (t == q) {
          const int4 raw = __ldg(reinterpret_cast<const int4*>(g.vtx + v));
          VtxInfo vi;
          vi.begin = ((unsigned long long)(unsigned)raw.y << 32) | (unsigned)raw.x;
          vi.deg = (unsigned)raw.z;
          vi.up = (unsigned)raw.w;
          bnd[t] = v;
          pb[t] = vi.begin;
          pe[t] = vi.begin + vi.deg;
          ha[t] = vi.begin + vi.up;
          hal[t] = v + 1;
          hb[t] = ha[t];
          hbl[t] = hal[t];
        }
    };

    // lower_bound(x) inside list q, bracketed by both hints; refreshes hint b
    auto lbq = [&](int q, uint32_t x) -> unsigned long long {
      unsigned long long r = 0;
#pragma unroll
      for (int t = 0; t < K; ++t)
        if (t == q) {
          unsigned long long lo = pb[t], hi = pe[t];
          if (x >= hal[t]) lo = max(lo, ha[t]); else hi = min(hi, ha[t]);
          if (x >= hbl[t]) lo = max(lo, hb[t]); else hi = min(hi, hb[t]);
          r = (x == hbl[t]) ? hb[t] : lower_bound_dev(nbr, lo, hi, x);
          hb[t] = r;
          hbl[t] = x;
        }
      return r;
    };

    // ------------------------------------------------ seed (ns_engine.cpp:29-33)
    if (alive) {
      const unsigned long long r0 = rng.next_below(g.arcs);
      const unsigned long long arc = __ldg(g.seed_arcs + r0);
      uint32_t u = (uint32_t)(arc >> 32), v = (uint32_t)arc;
      const bool swapped = p.seed_ordered && u > v;
      if (swapped) {
        uint32_t t = u;
        u = v;
        v = t;
      }
      bind(0, u);
      bind(1, v);
      nbound = 2;
      if (g.plain) {
        // arc r0 is nbr[r0] inside the source's list: a free lower_bound hint
        if (!swapped) {
          hb[0] = r0 + 1;
          hbl[0] = v + 1;
        } else {
          hb[1] = r0 + 1;
          hbl[1] = u + 1;
        }
      }
      if (COUNT_BYTES) bytes_acc += 64;
    }

    // ------------------------------------------------ steps (walker.hpp:30-83)
#pragma unroll
    for (int s = 0; s < K - 2; ++s) {
      const int j = s + 2;
      const unsigned in_m = p.in_mask[s], out_m = p.out_mask[s];
      const unsigned gt_m = p.gt_mask[s], lt_m = p.lt_mask[s];
      unsigned long long rs[K], re[K];
#pragma unroll
      for (int q = 0; q < K; ++q) rs[q] = re[q] = 0;
      int drv = -1;
      unsigned long long dsize = ~0ull;
      unsigned long long cnt = 0;
      unsigned long long mask = 0;
      int path = 0;  // 0 = dead/miss, 1 = single list, 2 = lane scan, 3 = warp
      uint32_t lo = 0, hi = 0xffffffffu;

      if (alive) {
#pragma unroll
        for (int q = 0; q < j; ++q) {
          if ((gt_m >> q) & 1u) lo = max(lo, bnd[q] + 1);
          if ((lt_m >> q) & 1u) hi = min(hi, bnd[q]);
        }
        int t_in = 0;
#pragma unroll
        for (int q = 0; q < j; ++q) {
          if ((in_m >> q) & 1u) {
            ++t_in;
            rs[q] = lo ? lbq(q, lo) : pb[q];
            re[q] = hi == 0xffffffffu ? pe[q] : lbq(q, hi);
            if (re[q] < rs[q]) re[q] = rs[q];
            const unsigned long long sz = re[q] - rs[q];
            if (sz < dsize) {
              dsize = sz;
              drv = q;
            }
          }
        }
        if (COUNT_BYTES) {
          used_mask |= in_m | out_m;
          if (t_in == 1 && out_m == 0) {
            bytes_acc += 32;
          } else {
#pragma unroll
            for (int q = 0; q < j; ++q) {
              if ((in_m >> q) & 1u) {
                const unsigned long long sp = sectors(rs[q], re[q]);
                bytes_acc += 32 * (q == drv ? sp : min(sp, dsize));
              } else if ((out_m >> q) & 1u) {
                bytes_acc += 32 * min(sectors(pb[q], pe[q]), dsize);
              }
            }
          }
        }
        if (dsize == 0) {
          path = 0;
        } else if (t_in == 1 && out_m == 0) {
          path = 1;
        } else if (dsize <= kSmallDriver) {
          path = 2;
        } else {
          path = 3;
        }
      }

      // ---------------- single list: count and pick by index arithmetic
      unsigned long long ex[K];
      if (path == 1) {
        unsigned long long a = 0, b = 0;
#pragma unroll
        for (int q = 0; q < j; ++q)
          if (q == drv) {
            a = rs[q];
            b = re[q];
          }
        unsigned long long excluded = 0;
#pragma unroll
        for (int q = 0; q < K; ++q) {
          ex[q] = ~0ull;
          if (q < j && bnd[q] >= lo && bnd[q] < hi) {
            const unsigned long long at = lower_bound_dev(nbr, a, b, bnd[q]);
            if (at < b && ldn(nbr, at) == bnd[q]) {
              ex[q] = at;
              ++excluded;
            }
          }
        }
        cnt = (b - a) - excluded;
      }

      // ---------------- short driver: lane-private scan
      if (path == 2) {
        unsigned long long dbeg = 0;
        unsigned long long cur[K];
#pragma unroll
        for (int q = 0; q < K; ++q) {
          cur[q] = rs[q];
          if (q == drv) dbeg = rs[q];
        }
        for (unsigned i = 0; i < dsize; ++i) {
          const uint32_t x = ldn(nbr, dbeg + i);
          bool ok = true;
          bool exhausted = false;
#pragma unroll
          for (int q = 0; q < j; ++q) {
            if (((in_m >> q) & 1u) && q != drv) {
              const unsigned long long c = gallop_dev(nbr, cur[q], re[q], x);
              cur[q] = c;
              if (c >= re[q]) {
                exhausted = true;
                ok = false;
              } else if (ldn(nbr, c) != x) {
                ok = false;
              }
            }
          }
#pragma unroll
          for (int q = 0; q < j; ++q) {
            if (ok && ((out_m >> q) & 1u)) {
              const unsigned long long at = lower_bound_dev(nbr, pb[q], pe[q], x);
              if (at < pe[q] && ldn(nbr, at) == x) ok = false;
            }
            if (x == bnd[q]) ok = false;
          }
          if (ok) mask |= 1ull << i;
          if (exhausted) break;
        }
        cnt = __popcll(mask);
      }

      // ---------------- long driver: the warp intersects for one lane at a time
      uint32_t coop_pick = 0;
      unsigned long long coop_at = 0;
      unsigned pend = __ballot_sync(FULL, path == 3);
      while (pend) {
        const int L = __ffs(pend) - 1;
        pend &= pend - 1;
        uint32_t cb[K];
        unsigned long long crs[K], cre[K], cpb[K], cpe[K];
#pragma unroll
        for (int q = 0; q < K; ++q) {
          cb[q] = __shfl_sync(FULL, bnd[q], L);
          crs[q] = __shfl_sync(FULL, rs[q], L);
          cre[q] = __shfl_sync(FULL, re[q], L);
          cpb[q] = __shfl_sync(FULL, pb[q], L);
          cpe[q] = __shfl_sync(FULL, pe[q], L);
        }
        const int cdrv = __shfl_sync(FULL, drv, L);
        const unsigned long long cds = __shfl_sync(FULL, dsize, L);
        unsigned long long dbeg = 0;
#pragma unroll
        for (int q = 0; q < K; ++q)
          if (q == cdrv) dbeg = crs[q];
        const unsigned long long nch = (cds + 31) >> 5;

        // one pass over driver chunks; returns total hits, stages ballots
        auto chunk_ballot = [&](unsigned long long c, unsigned long long* ccur) -> unsigned {
          const unsigned long long i = c * 32 + lane;
          const bool valid = i < cds;
          const uint32_t x = valid ? ldn(nbr, dbeg + i) : 0xffffffffu;
          bool ok = valid;
          const int last = (int)min(31ull, cds - 1 - c * 32);
#pragma unroll
          for (int q = 0; q < j; ++q) {
            if (((in_m >> q) & 1u) && q != cdrv) {
              const unsigned long long at = lower_bound_dev(nbr, ccur[q], cre[q], x);
              if (!(at < cre[q] && ldn(nbr, at) == x)) ok = false;
              ccur[q] = __shfl_sync(FULL, at, last);
            }
          }
#pragma unroll
          for (int q = 0; q < j; ++q) {
            if (ok && ((out_m >> q) & 1u)) {
              const unsigned long long at = lower_bound_dev(nbr, cpb[q], cpe[q], x);
              if (at < cpe[q] && ldn(nbr, at) == x) ok = false;
            }
            if (x == cb[q]) ok = false;
          }
          return __ballot_sync(FULL, ok);
        };

        unsigned long long ccur[K];
#pragma unroll
        for (int q = 0; q < K; ++q) ccur[q] = crs[q];
        unsigned long long total = 0;
        for (unsigned long long c = 0; c < nch; ++c) {
          const unsigned bal = chunk_ballot(c, ccur);
          if (c < kBallotWords && lane == 0) ballots[c] = bal;
          total += __popc(bal);
        }
        __syncwarp();
        // lane L consumes its next draw exactly as the reference would
        unsigned long long r = 0;
        if (lane == L && total > 0) r = rng.next_below(total);
        r = __shfl_sync(FULL, r, L);
        if (total > 0) {
          unsigned long long hit_index = 0;  // index within the driver
          if (nch <= kBallotWords) {
            unsigned long long before = 0;
            bool found = false;
            for (int half = 0; half < 2 && !found; ++half) {
              const int w = half * 32 + lane;
              const unsigned word = (unsigned long long)w < nch ? ballots[w] : 0u;
              unsigned incl = __popc(word);
#pragma unroll
              for (int d = 1; d < 32; d <<= 1) {
                const unsigned o = __shfl_up_sync(FULL, incl, d);
                if (lane >= d) incl += o;
              }
              const unsigned excl = incl - __popc(word);
              const bool mine = before + excl <= r && r < before + incl;
              const unsigned who = __ballot_sync(FULL, mine);
              if (who) {
                const int src = __ffs(who) - 1;
                unsigned long long hi_idx = 0;
                if (lane == src) hi_idx = (unsigned long long)w * 32 + __fns(word, 0, (int)(r - before - excl) + 1);
                hit_index = __shfl_sync(FULL, hi_idx, src);
                found = true;
              }
              before += __shfl_sync(FULL, incl, 31);
            }
          } else {
#pragma unroll
            for (int q = 0; q < K; ++q) ccur[q] = crs[q];
            unsigned long long before = 0;
            for (unsigned long long c = 0; c < nch; ++c) {
              const unsigned bal = chunk_ballot(c, ccur);
              const unsigned pc = __popc(bal);
              if (r < before + pc) {
                hit_index = c * 32 + __fns(bal, 0, (int)(r - before) + 1);
                break;
              }
              before += pc;
            }
          }
          if (lane == L) {
            coop_at = dbeg + hit_index;
            coop_pick = ldn(nbr, coop_at);
          }
        }
        if (lane == L) cnt = total;
        __syncwarp();
      }

      // ---------------- finalize the step for this lane
      if (alive) {
        if (cnt == 0) {
          alive = false;  // miss: early break (ns_engine.cpp:38)
        } else {
          alpha = __dmul_rn(alpha, (double)cnt);
          uint32_t pick = 0;
          unsigned long long at = 0;
          if (path == 1) {
            const unsigned long long r = rng.next_below(cnt);
            unsigned long long a = 0;
#pragma unroll
            for (int q = 0; q < j; ++q)
              if (q == drv) a = rs[q];
            at = a + r;
            for (int it = 0; it < K; ++it) {  // skip excluded positions <= at
              unsigned long long c = 0;
#pragma unroll
              for (int q = 0; q < K; ++q) c += (ex[q] <= at) ? 1 : 0;
              const unsigned long long nat = a + r + c;
              if (nat == at) break;
              at = nat;
            }
            pick = ldn(nbr, at);
          } else if (path == 2) {
            const unsigned long long r = rng.next_below(cnt);
            unsigned long long dbeg = 0;
#pragma unroll
            for (int q = 0; q < j; ++q)
              if (q == drv) dbeg = rs[q];
            at = dbeg + nth_bit64(mask, (int)r);
            pick = ldn(nbr, at);
          } else {
            at = coop_at;
            pick = coop_pick;
          }
          bind(j, pick);
          nbound = j + 1;
          // the pick sits at `at` in the driver's list: lower_bound(pick+1) = at+1
#pragma unroll
          for (int q = 0; q < j; ++q)
            if (q == drv) {
              hb[q] = at + 1;
              hbl[q] = pick + 1;
            }
        }
      }
    }

    if (idx < count) {
      values[idx] = alive ? alpha : 0.0;
      if (bindings) {
#pragma unroll
        for (int q = 0; q < K; ++q) bindings[idx * K + q] = q < nbound ? bnd[q] : 0xffffffffu;
      }
      if (COUNT_BYTES) bytes_acc += 32ull * __popc(used_mask);
    }
  }
  if (COUNT_BYTES) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) bytes_acc += __shfl_xor_sync(FULL, bytes_acc, d);
    if (lane == 0) atomicAdd(bytes_out, bytes_acc);
  }
}

// ------------------------------------------------------------ moments / convergence
// One warp per window; fixed-shape shuffle tree => deterministic partials.
__global__ void window_moments_kernel(const double* __restrict__ v, unsigned long long count,
                                      unsigned long long window, agpm_accumulator* __restrict__ out,
                                      unsigned long long nwin) {
  const int lane = threadIdx.x & 31;
  const unsigned long long w0 = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
  const unsigned long long nw = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
  for (unsigned long long w = w0; w < nwin; w += nw) {
    const unsigned long long b = w * window;
    const unsigned long long e = min(count, b + window);
    unsigned long long n = 0, hits = 0;
    double s = 0.0, sq = 0.0;
    for (unsigned long long i = b + lane; i < e; i += 32) {
      const double x = v[i];
      ++n;
      hits += x != 0.0;
      s = __dadd_rn(s, x);
      sq = __dadd_rn(sq, __dmul_rn(x, x));
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      n += __shfl_xor_sync(FULL, n, d);
      hits += __shfl_xor_sync(FULL, hits, d);
      s = __dadd_rn(s, __shfl_xor_sync(FULL, s, d));
      sq = __dadd_rn(sq, __shfl_xor_sync(FULL, sq, d));
    }
    if (lane == 0) out[w] = agpm_accumulator{n, hits, s, sq};
  }
}

struct OnlineState {
  agpm_accumulator acc;
  agpm_report rep;
  unsigned long long windows;
  int stopped;
  int pad;
};

// stats.cpp:57-70 with the reference's operation order, no FMA contraction
__device__ agpm_report predicted_error_dev(const agpm_accumulator& a, double z) {
  agpm_report r;
  r.mu = 0.0;
  r.sigma = 0.0;
  r.epsilon_hat = __longlong_as_double(0x7ff0000000000000ll);
  r.n = a.n;
  r.converged = 0;
  r.hit_rate = 0.0;
  if (a.n == 0) return r;
  const double n = (double)a.n;
  r.hit_rate = __ddiv_rn((double)a.hits, n);
  r.mu = __ddiv_rn(a.sum, n);
  if (!(a.sum > 0.0) || a.n < 2) return r;
  double var = __dsub_rn(__ddiv_rn(a.squared_sum, n), __dmul_rn(r.mu, r.mu));
  if (var < 0.0) var = 0.0;
  r.sigma = __dsqrt_rn(__ddiv_rn(var, n));
  r.epsilon_hat = __ddiv_rn(__dmul_rn(z, r.sigma), r.mu);
  return r;
}

// Sequential merge of window partials in window order (ns_engine.cpp:121-137)
__global__ void converge_kernel(const agpm_accumulator* __restrict__ win, unsigned long long nwin,
                                OnlineState* st, double z, double eps, unsigned long long max_samples) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  OnlineState s = *st;
  for (unsigned long long w = 0; w < nwin && !s.stopped; ++w) {
    const agpm_accumulator a = win[w];
    s.acc.n += a.n;
    s.acc.hits += a.hits;
    s.acc.sum = __dadd_rn(s.acc.sum, a.sum);
    s.acc.squared_sum = __dadd_rn(s.acc.squared_sum, a.squared_sum);
    ++s.windows;
    s.rep = predicted_error_dev(s.acc, z);
    if (s.rep.epsilon_hat <= eps) {
      s.rep.converged = 1;
      s.stopped = 1;
    } else if (s.acc.n >= max_samples) {
      s.stopped = 1;
    }
  }
  *st = s;
}

// ------------------------------------------------------------ host side
namespace {

DevPlan make_dev_plan(const agpm_graph* g, const agpm_plan* plan) {
  if (!plan) throw std::invalid_argument("null plan");
  if (plan->k < 2 || plan->k > AGPM_MAX_K || plan->n_steps != plan->k - 2)
    throw std::invalid_argument("malformed plan");
  if (plan->verify_mode != 0)
    throw std::invalid_argument("the device sampler implements eager verification (VerifyMode::Eager)");
  if (g->edge_count == 0) throw std::invalid_argument("cannot sample from an empty graph");
  if (g->oriented) throw std::invalid_argument("sampling runs on the symmetric graph");
  DevPlan d{};
  d.k = plan->k;
  d.n_steps = plan->n_steps;
  d.seed_ordered = plan->seed_ordered;
  d.alpha0 = plan->seed_ordered ? static_cast<double>(g->edge_count) : 2.0 * static_cast<double>(g->edge_count);
  for (int s = 0; s < plan->n_steps; ++s) {
    const agpm_plan_step& st = plan->steps[s];
    unsigned in = 0, out = 0, gt = 0, lt = 0;
    for (int i = 0; i < st.n_in; ++i) in |= 1u << st.in_positions[i];
    for (int i = 0; i < st.n_out; ++i) out |= 1u << st.out_positions[i];
    for (int i = 0; i < st.n_gt; ++i) gt |= 1u << st.greater_than[i];
    for (int i = 0; i < st.n_lt; ++i) lt |= 1u << st.less_than[i];
    if (in == 0 || (in >> (s + 2)) || (out >> (s + 2)) || (gt >> (s + 2)) || (lt >> (s + 2)))
      throw std::invalid_argument("malformed plan step");
    d.in_mask[s] = (unsigned short)in;
    d.out_mask[s] = (unsigned short)out;
    d.gt_mask[s] = (unsigned short)gt;
    d.lt_mask[s] = (unsigned short)lt;
  }
  return d;
}

GraphArgs graph_args(const agpm_graph* g) {
  GraphArgs a;
  a.vtx = g->vtx;
  a.nbr = g->nbr;
  a.seed_arcs = g->seed_arcs;
  a.arcs = g->arcs;
  a.plain = g->plain;
  return a;
}

template <int K, bool CB>
void launch_k(const GraphArgs& ga, const DevPlan& dp, uint64_t seed, uint64_t first, uint64_t count,
              double* values, uint32_t* bindings, unsigned long long* cursor, unsigned long long* bytes,
              cudaStream_t s) {
  DeviceCtx& ctx = ctx_for_current_device();
  static int occ = -1;
  if (occ < 0) {
    int o = 0;
    AGPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, ns_sample_kernel<K, CB>, kThreads, 0));
    occ = o > 0 ? o : 1;
  }
  const uint64_t warps_needed = (count + 31) / 32;
  uint64_t blocks = std::min<uint64_t>((uint64_t)ctx.sm_count * occ, (warps_needed + kWarps - 1) / kWarps);
  if (blocks == 0) blocks = 1;
  ns_sample_kernel<K, CB><<<(unsigned)blocks, kThreads, 0, s>>>(ga, dp, seed, first, count, values,
                                                                bindings, cursor, bytes);
  count_launch();
  AGPM_CUDA(cudaGetLastError());
}

// enqueue one sampling launch for ids [first, first+count) into d_values
void enqueue_sample(const agpm_graph* g, const DevPlan& dp, uint64_t seed, uint64_t first, uint64_t count,
                    double* d_values, uint32_t* d_bindings, unsigned long long* d_bytes, cudaStream_t s) {
  DeviceCtx& ctx = ctx_for_current_device();
  auto* cursor = static_cast<unsigned long long*>(ctx.get(0, 64));
  AGPM_CUDA(cudaMemsetAsync(cursor, 0, sizeof(unsigned long long), s));
  const GraphArgs ga = graph_args(g);
  const bool cb = d_bytes != nullptr;
#define AGPM_K(KK)                                                                              \
  case KK:                                                                                      \
    if (cb)                                                                                     \
      launch_k<KK, true>(ga, dp, seed, first, count, d_values, d_bindings, cursor, d_bytes, s); \
    else                                                                                        \
      launch_k<KK, false>(ga, dp, seed, first, count, d_values, d_bindings, cursor, d_bytes, s); \
    break;
  switch (dp.k) {
    AGPM_K(3)
    AGPM_K(4)
    AGPM_K(5)
    AGPM_K(6)
    AGPM_K(7)
    AGPM_K(8)
    AGPM_K(9)
    default:
      throw std::invalid_argument("device sampler needs 3 <= k <= 9");
  }
#undef AGPM_K
}

void enqueue_moments(const double* d_values, uint64_t count, uint64_t window, agpm_accumulator* d_out,
                     cudaStream_t s) {
  DeviceCtx& ctx = ctx_for_current_device();
  const uint64_t nwin = (count + window - 1) / window;
  if (nwin == 0) return;
  uint64_t blocks = std::min<uint64_t>((nwin + 7) / 8, (uint64_t)ctx.sm_count * 8);
  window_moments_kernel<<<(unsigned)blocks, 256, 0, s>>>(d_values, count, window, d_out, nwin);
  count_launch();
  AGPM_CUDA(cudaGetLastError());
}

constexpr uint64_t kChunk = 1ull << 24;

}  // namespace

}  // namespace agpm_b200

using namespace agpm_b200;

extern "C" {

int agpm_ns_sample_dev(agpm_graph* g, const agpm_plan* plan, uint64_t seed, uint64_t first_id,
                       uint64_t count, double* d_values, void* stream) {
  return guarded([&] {
    const DevPlan dp = make_dev_plan(g, plan);
    if (count) enqueue_sample(g, dp, seed, first_id, count, d_values, nullptr, nullptr, pick_stream(stream));
  });
}

int agpm_window_moments_dev(const double* d_values, uint64_t count, uint64_t window,
                            agpm_accumulator* d_out, void* stream) {
  return guarded([&] {
    if (window == 0) throw std::invalid_argument("window must be >= 1");
    enqueue_moments(d_values, count, window, d_out, pick_stream(stream));
  });
}

int agpm_ns_draw(agpm_graph* g, const agpm_plan* plan, uint64_t seed, uint64_t first_id, uint64_t count,
                 double* values, uint8_t* hits, uint32_t* bindings, void* stream) {
  return guarded([&] {
    const DevPlan dp = make_dev_plan(g, plan);
    DeviceCtx& ctx = ctx_for_current_device();
    cudaStream_t s = pick_stream(stream);
    const uint64_t chunk = std::min<uint64_t>(count ? count : 1, kChunk);
    auto* d_values = static_cast<double*>(ctx.get(1, sizeof(double) * chunk));
    uint32_t* d_bind = bindings ? static_cast<uint32_t*>(ctx.get(2, sizeof(uint32_t) * chunk * dp.k)) : nullptr;
    for (uint64_t done = 0; done < count; done += chunk) {
      const uint64_t c = std::min(chunk, count - done);
      enqueue_sample(g, dp, seed, first_id + done, c, d_values, d_bind, nullptr, s);
      AGPM_CUDA(cudaMemcpyAsync(values + done, d_values, sizeof(double) * c, cudaMemcpyDeviceToHost, s));
      if (bindings)
        AGPM_CUDA(cudaMemcpyAsync(bindings + done * dp.k, d_bind, sizeof(uint32_t) * c * dp.k,
                                  cudaMemcpyDeviceToHost, s));
      AGPM_CUDA(cudaStreamSynchronize(s));
      if (hits)
        for (uint64_t i = 0; i < c; ++i) hits[done + i] = values[done + i] != 0.0;
    }
  });
}

int agpm_ns_bmin_bytes(agpm_graph* g, const agpm_plan* plan, uint64_t seed, uint64_t first_id,
                       uint64_t count, uint64_t* total_bytes, void* stream) {
  return guarded([&] {
    const DevPlan dp = make_dev_plan(g, plan);
    DeviceCtx& ctx = ctx_for_current_device();
    cudaStream_t s = pick_stream(stream);
    const uint64_t chunk = std::min<uint64_t>(count ? count : 1, kChunk);
    auto* d_values = static_cast<double*>(ctx.get(1, sizeof(double) * chunk));
    auto* d_bytes = static_cast<unsigned long long*>(ctx.get(3, 64));
    AGPM_CUDA(cudaMemsetAsync(d_bytes, 0, 8, s));
    for (uint64_t done = 0; done < count; done += chunk) {
      const uint64_t c = std::min(chunk, count - done);
      enqueue_sample(g, dp, seed, first_id + done, c, d_values, nullptr, d_bytes, s);
    }
    unsigned long long h = 0;
    AGPM_CUDA(cudaMemcpyAsync(&h, d_bytes, 8, cudaMemcpyDeviceToHost, s));
    AGPM_CUDA(cudaStreamSynchronize(s));
    *total_bytes = h;
  });
}

int agpm_ns_fixed_budget(agpm_graph* g, const agpm_plan* plan, uint64_t budget, uint64_t seed,
                         agpm_accumulator* out, void* stream) {
  // run_fixed_budget (ns_engine.cpp:142-153): one window of `budget` samples
  return guarded([&] {
    if (budget < 1) throw std::invalid_argument("sample budget must be >= 1");
    const DevPlan dp = make_dev_plan(g, plan);
    DeviceCtx& ctx = ctx_for_current_device();
    cudaStream_t s = pick_stream(stream);
    const uint64_t chunk = std::min<uint64_t>(budget, kChunk);
    constexpr uint64_t kWin = 4096;
    const uint64_t nwin_chunk = (chunk + kWin - 1) / kWin;
    auto* d_values = static_cast<double*>(ctx.get(1, sizeof(double) * chunk));
    auto* d_win = static_cast<agpm_accumulator*>(ctx.get(4, sizeof(agpm_accumulator) * nwin_chunk));
    auto* h_win = static_cast<agpm_accumulator*>(ctx.get_pinned(sizeof(agpm_accumulator) * nwin_chunk));
    agpm_accumulator acc{0, 0, 0.0, 0.0};
    for (uint64_t done = 0; done < budget; done += chunk) {
      const uint64_t c = std::min(chunk, budget - done);
      const uint64_t nw = (c + kWin - 1) / kWin;
      enqueue_sample(g, dp, seed, done, c, d_values, nullptr, nullptr, s);
      enqueue_moments(d_values, c, kWin, d_win, s);
      AGPM_CUDA(cudaMemcpyAsync(h_win, d_win, sizeof(agpm_accumulator) * nw, cudaMemcpyDeviceToHost, s));
      AGPM_CUDA(cudaStreamSynchronize(s));
      for (uint64_t w = 0; w < nw; ++w) {
        acc.n += h_win[w].n;
        acc.hits += h_win[w].hits;
        acc.sum += h_win[w].sum;
        acc.squared_sum += h_win[w].squared_sum;
      }
    }
    *out = acc;
  });
}

int agpm_ns_online(agpm_graph* g, const agpm_plan* plan, double eps, double delta,
                   const agpm_online_policy* policy, uint64_t seed, agpm_online_result* out,
                   void* stream) {
  // run_ns_online (ns_engine.cpp:106-140) with workers = 1: windows of
  // W = max(n_min, 10) (or >= profiled/10) samples; convergence is evaluated
  // after EVERY window even though the device draws speculative batches of
  // many windows, so the stop n equals the reference's.
  return guarded([&] {
    if (!(eps > 0.0) || !(eps < 1.0)) throw std::invalid_argument("error bound must be inside (0,1)");
    if (!(delta > 0.0) || !(delta < 1.0)) throw std::invalid_argument("delta must be inside (0,1)");
    const DevPlan dp = make_dev_plan(g, plan);
    agpm_online_policy pol = policy ? *policy : agpm_online_policy{1000, 1000000000ull, 0};
    DeviceCtx& ctx = ctx_for_current_device();
    cudaStream_t s = pick_stream(stream);
    const double z = inv_norm_cdf(1.0 - delta / 2.0);
    uint64_t window = std::max<uint64_t>(pol.n_min, 10);
    if (pol.profiled_n_samples > 0) window = std::max(window, pol.profiled_n_samples / 10);
    const uint64_t max_batch = std::max<uint64_t>(window, (kChunk / window) * window);
    uint64_t batch = std::min(max_batch, std::max<uint64_t>(window, ((1ull << 16) / window) * window));

    auto* d_values = static_cast<double*>(ctx.get(1, sizeof(double) * max_batch));
    auto* d_win = static_cast<agpm_accumulator*>(ctx.get(4, sizeof(agpm_accumulator) * (max_batch / window + 1)));
    auto* d_state = static_cast<OnlineState*>(ctx.get(5, sizeof(OnlineState)));
    auto* h_state = static_cast<OnlineState*>(ctx.get_pinned(sizeof(OnlineState)));
    AGPM_CUDA(cudaMemsetAsync(d_state, 0, sizeof(OnlineState), s));
    auto t0 = std::chrono::steady_clock::now();
    uint64_t launched = 0;
    std::memset(h_state, 0, sizeof(OnlineState));
    while (launched < pol.max_samples) {
      const uint64_t c = std::min(batch, pol.max_samples - launched);
      const uint64_t nw = (c + window - 1) / window;
      enqueue_sample(g, dp, seed, launched, c, d_values, nullptr, nullptr, s);
      enqueue_moments(d_values, c, window, d_win, s);
      converge_kernel<<<1, 32, 0, s>>>(d_win, nw, d_state, z, eps, pol.max_samples);
      count_launch();
      AGPM_CUDA(cudaGetLastError());
      AGPM_CUDA(cudaMemcpyAsync(h_state, d_state, sizeof(OnlineState), cudaMemcpyDeviceToHost, s));
      AGPM_CUDA(cudaStreamSynchronize(s));
      launched += c;
      if (h_state->stopped) break;
      batch = std::min(max_batch, batch * 2);
    }
    auto t1 = std::chrono::steady_clock::now();
    std::memset(out, 0, sizeof(*out));
    out->report = h_state->rep;
    out->accumulator = h_state->acc;
    out->windows = h_state->windows;
    out->samples_launched = launched;
    out->seconds = std::chrono::duration<double>(t1 - t0).count();
  });
}

}  // extern "C"
