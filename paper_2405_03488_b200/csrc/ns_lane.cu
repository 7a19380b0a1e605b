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
#include <stdexcept>
#include <chrono>
#include <cmath>
#include <cstring>
#include <vector>

#include "ns_common.cuh"

namespace agpm_b200 {
namespace {

constexpr int kSmallDriver = 64;   // lane-private scan up to this many driver elements

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


template <int K, bool CB>
void launch_k(const SampleLaunch& L, cudaStream_t s) {
  DeviceCtx& ctx = ctx_for_current_device();
  static int occ = -1;
  if (occ < 0) {
    int o = 0;
    AGPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, ns_sample_kernel<K, CB>, kThreads, 0));
    occ = o > 0 ? o : 1;
  }
  const uint64_t warps_needed = (L.count + 31) / 32;
  uint64_t blocks = std::min<uint64_t>((uint64_t)ctx.sm_count * occ, (warps_needed + kWarps - 1) / kWarps);
  if (blocks == 0) blocks = 1;
  ns_sample_kernel<K, CB><<<(unsigned)blocks, kThreads, 0, s>>>(L.g, L.p, L.seed, L.first_id, L.count, L.values,
                                                                L.bindings, L.cursor, L.bytes_out);
  count_launch();
  AGPM_CUDA(cudaGetLastError());
}

}  // namespace

void launch_ns_lane(const SampleLaunch& L, cudaStream_t s) {
  const bool cb = L.bytes_out != nullptr;
#define AGPM_K(KK)                   \
  case KK:                           \
    if (cb)                          \
      launch_k<KK, true>(L, s);      \
    else                             \
      launch_k<KK, false>(L, s);     \
    break;
  switch (L.p.k) {
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

}  // namespace agpm_b200
