// Warp-cooperative eager-verify sampler: ONE warp per sample.
//
// Every lane holds an identical copy of the sample state (bindings, list
// bounds, CounterRng(seed, 0, id)), so every RNG draw, branch and pick is
// warp-uniform; lanes only split the memory work:
//   * k-ary search — lower_bound over a sorted adjacency range probes 32
//     positions at once (one independent load per lane, one ballot), so a
//     30k-element hub list resolves in 3 dependent rounds instead of 15;
//   * chunk intersection — the driver (smallest bound-restricted in-list) is
//     read 32 elements per coalesced load; each other in-list is streamed in
//     32-element chunks over the same value window and membership is a
//     5-step shuffle search across lanes; windows far ahead are skipped with
//     the k-ary search, so cost follows min(merge, search) per list;
//   * ballots of the hit mask go to shared memory so the r-th candidate is
//     found with a popcount prefix, not a second intersection pass.
// The candidate set is S = (∩ in-lists) \ (∪ out-lists) \ bound vertices,
// restricted to [lo, hi) by the step's order constraints — exactly
// build_step_candidates (walker.hpp:30-83) — enumerated ascending, and the
// pick is S[next_below(|S|)] (ns_engine.cpp:36-40): per-sample results are
// bit-identical to the reference's draw_sample with workers = 1.
#include <algorithm>
#include <stdexcept>

#include "ns_common.cuh"

namespace agpm_b200 {
namespace {

constexpr uint32_t INF = 0xffffffffu;
constexpr int kWarpBatch = 8;  // sample ids claimed per cursor atomic

template <int K, bool COUNT_BYTES>
__global__ void __launch_bounds__(kThreads) ns_warp_kernel(const SampleLaunch L) {
  __shared__ uint32_t s_ballot[kWarps][kBallotWords];
  const int lane = threadIdx.x & 31;
  uint32_t* ballots = s_ballot[threadIdx.x >> 5];
  const uint32_t* __restrict__ nbr = L.g.nbr;
  const DevPlan& p = L.p;
  unsigned long long bytes_acc = 0;
  unsigned long long next = 0, end = 0;

  for (;;) {
    if (next >= end) {
      unsigned long long b = 0;
      if (lane == 0) b = atomicAdd(L.cursor, (unsigned long long)kWarpBatch);
      b = __shfl_sync(FULL, b, 0);
      if (b >= L.count) break;
      next = b;
      end = min(L.count, b + kWarpBatch);
    }
    const unsigned long long idx = next++;
    CounterRng rng(L.seed, 0, L.first_id + idx);

    // per-position state (warp-uniform). Offsets are relative to pb[q].
    uint32_t bnd[K], pd[K], up[K], hbo[K], hbl[K];
    unsigned long long pb[K];
#pragma unroll
    for (int q = 0; q < K; ++q) {
      bnd[q] = INF;
      pd[q] = up[q] = hbo[q] = hbl[q] = 0;
      pb[q] = 0;
    }
    auto bind = [&](int q, uint32_t v) {
      const VtxInfo vi = load_vtx(L.g.vtx, v);
#pragma unroll
      for (int t = 0; t < K; ++t)
        if (t == q) {
          bnd[t] = v;
          pb[t] = vi.begin;
          pd[t] = vi.deg;
          up[t] = vi.up;  // lower_bound(v + 1) = up
          hbo[t] = vi.up;
          hbl[t] = v + 1;
        }
    };
    // lower_bound(x) in list q bracketed by its two hints; update refreshes hint b
    auto lbq = [&](int q, uint32_t x, bool update) -> uint32_t {
      uint32_t r = 0;
#pragma unroll
      for (int t = 0; t < K; ++t)
        if (t == q) {
          uint32_t lo = 0, hi = pd[t];
          if (x >= bnd[t] + 1) lo = max(lo, up[t]); else hi = min(hi, up[t]);
          if (x >= hbl[t]) lo = max(lo, hbo[t]); else hi = min(hi, hbo[t]);
          r = x == hbl[t] ? hbo[t] : kary_lb(nbr + pb[t], lo, hi, x, lane, nullptr);
          if (update) {
            hbo[t] = r;
            hbl[t] = x;
          }
        }
      return r;
    };

    double alpha = p.alpha0;
    bool alive = true;
    int nbound = 2;
    unsigned used_mask = 0;

    // ------------------------------------------------ seed (ns_engine.cpp:29-33)
    {
      const unsigned long long r0 = rng.next_below(L.g.arcs);
      const unsigned long long arc = __ldg(L.g.seed_arcs + r0);
      uint32_t u = (uint32_t)(arc >> 32), v = (uint32_t)arc;
      const bool swapped = p.seed_ordered && u > v;
      if (swapped) {
        const uint32_t t = u;
        u = v;
        v = t;
      }
      bind(0, u);
      bind(1, v);
      if (L.g.plain) {  // arc r0 = nbr[r0] inside its source's list
        if (!swapped) {
          hbo[0] = (uint32_t)(r0 - pb[0]) + 1;
          hbl[0] = v + 1;
        } else {
          hbo[1] = (uint32_t)(r0 - pb[1]) + 1;
          hbl[1] = u + 1;
        }
      }
      if (COUNT_BYTES) bytes_acc += 64;
    }

    // ------------------------------------------------ steps (walker.hpp:30-83)
#pragma unroll
    for (int s = 0; s < K - 2; ++s) {
      if (!alive) break;
      const int j = s + 2;
      const unsigned in_m = p.in_mask[s], out_m = p.out_mask[s];
      const unsigned gt_m = p.gt_mask[s], lt_m = p.lt_mask[s];
      uint32_t lo = 0, hi = INF;
#pragma unroll
      for (int q = 0; q < j; ++q) {
        if ((gt_m >> q) & 1u) lo = max(lo, bnd[q] + 1);
        if ((lt_m >> q) & 1u) hi = min(hi, bnd[q]);
      }
      uint32_t rs[K], re[K];
      int drv = -1, t_in = 0;
      uint32_t dsize = INF;
#pragma unroll
      for (int q = 0; q < K; ++q) {
        rs[q] = re[q] = 0;
        if (q < j && ((in_m >> q) & 1u)) {
          ++t_in;
          rs[q] = lo ? lbq(q, lo, true) : 0;
          re[q] = hi == INF ? pd[q] : lbq(q, hi, false);
          if (re[q] < rs[q]) re[q] = rs[q];
          if (re[q] - rs[q] < dsize) {
            dsize = re[q] - rs[q];
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
              const unsigned long long sp = sectors(pb[q] + rs[q], pb[q] + re[q]);
              bytes_acc += 32 * (q == drv ? sp : min(sp, (unsigned long long)dsize));
            } else if ((out_m >> q) & 1u) {
              bytes_acc += 32 * min(sectors(pb[q], pb[q] + pd[q]), (unsigned long long)dsize);
            }
          }
        }
      }
      unsigned long long dbase = 0;  // absolute index of the driver range start
#pragma unroll
      for (int q = 0; q < K; ++q)
        if (q == drv) dbase = pb[q] + rs[q];

      unsigned long long cnt = 0, at = 0;  // |S| and absolute index of the pick
      if (dsize == 0) {
        alive = false;
      } else if (t_in == 1 && out_m == 0) {
        // ---------------- single list: |S| = |range| - bound vertices inside it
        uint32_t ex[K];
        uint32_t nex = 0;
#pragma unroll
        for (int q = 0; q < K; ++q) {
          ex[q] = INF;
          if (q < j && bnd[q] >= lo && bnd[q] < hi) {
            bool f = false;
            const uint32_t o = kary_lb(nbr + dbase, 0, dsize, bnd[q], lane, &f);
            if (f) {
              ex[q] = o;
              ++nex;
            }
          }
        }
        cnt = dsize - nex;
        if (cnt == 0) {
          alive = false;
        } else {
          const uint32_t r = (uint32_t)rng.next_below(cnt);
          uint32_t o = r;
          for (int it = 0; it < K; ++it) {  // skip excluded offsets <= o
            uint32_t c = 0;
#pragma unroll
            for (int q = 0; q < K; ++q) c += ex[q] <= o ? 1u : 0u;
            if (r + c == o) break;
            o = r + c;
          }
          at = dbase + o;
        }
      } else {
        // ---------------- chunked intersection of the driver with the other lists
        uint32_t cur[K];
        bool exhausted = false;
        auto chunk = [&](uint32_t ia) -> unsigned {
          const uint32_t i = ia + lane;
          const bool valid = i < dsize;
          const uint32_t a = valid ? ldn(nbr, dbase + i) : INF;
          const int last = (int)min(31u, dsize - 1 - ia);
          const uint32_t a_last = __shfl_sync(FULL, a, last);
          bool ok = valid;
#pragma unroll
          for (int q = 0; q < K; ++q) {
            if (q < j && ((in_m >> q) & 1u) && q != drv) {
              const uint32_t* B = nbr + pb[q];
              const uint32_t c = cur[q];
              const uint32_t e = re[q];
              bool hit = false;
              if (c >= e) {  // list q exhausted: no driver element from here on matches
                exhausted = true;
              } else if (e - c <= 32) {  // whole remaining window in one coalesced chunk
                const uint32_t b = c + lane < e ? ldn(B, c + lane) : INF;
                hit = chunk_contains(b, a);
                cur[q] = c + __popc(__ballot_sync(FULL, b <= a_last));
              } else {  // per-lane search; the cursor follows the chunk's last element
                const uint32_t o = c + lane_lb(B + c, e - c, a);
                hit = o < e && ldn(B, o) == a;
                cur[q] = __shfl_sync(FULL, o, last);
              }
              ok = ok && hit;
            }
          }
#pragma unroll
          for (int q = 0; q < K; ++q) {
            if (q < j) {
              if (ok && ((out_m >> q) & 1u)) {
                const unsigned long long o = lower_bound_dev(nbr, pb[q], pb[q] + pd[q], a);
                if (o < pb[q] + pd[q] && ldn(nbr, o) == a) ok = false;
              }
              if (a == bnd[q]) ok = false;
            }
          }
          return __ballot_sync(FULL, ok);
        };

#pragma unroll
        for (int q = 0; q < K; ++q) cur[q] = rs[q];
        const uint32_t nch = (dsize + 31) >> 5;
        uint32_t done = 0;
        for (uint32_t c = 0; c < nch && !exhausted; ++c) {
          const unsigned bal = chunk(c * 32);
          if (c < kBallotWords && lane == 0) ballots[c] = bal;
          cnt += __popc(bal);
          done = c + 1;
        }
        __syncwarp();
        if (cnt == 0) {
          alive = false;
        } else {
          const unsigned long long r = rng.next_below(cnt);
          uint32_t hit_index = 0;
          if (done <= kBallotWords) {
            unsigned long long before = 0;
            for (int half = 0; half < 2; ++half) {
              const uint32_t w = half * 32 + lane;
              const unsigned word = w < done ? ballots[w] : 0u;
              unsigned incl = __popc(word);
#pragma unroll
              for (int d = 1; d < 32; d <<= 1) {
                const unsigned o = __shfl_up_sync(FULL, incl, d);
                if (lane >= d) incl += o;
              }
              const unsigned excl = incl - __popc(word);
              const unsigned who = __ballot_sync(FULL, before + excl <= r && r < before + incl);
              if (who) {
                const int src = __ffs(who) - 1;
                uint32_t hi_idx = 0;
                if (lane == src) hi_idx = w * 32 + __fns(word, 0, (int)(r - before - excl) + 1);
                hit_index = __shfl_sync(FULL, hi_idx, src);
                break;
              }
              before += __shfl_sync(FULL, incl, 31);
            }
          } else {  // driver longer than the staged ballots: replay until the r-th hit
#pragma unroll
            for (int q = 0; q < K; ++q) cur[q] = rs[q];
            exhausted = false;
            unsigned long long before = 0;
            for (uint32_t c = 0; c < nch; ++c) {
              const unsigned bal = chunk(c * 32);
              const unsigned pc = __popc(bal);
              if (r < before + pc) {
                hit_index = c * 32 + __fns(bal, 0, (int)(r - before) + 1);
                break;
              }
              before += pc;
            }
          }
          at = dbase + hit_index;
        }
        __syncwarp();
      }

      if (alive) {
        alpha = __dmul_rn(alpha, (double)cnt);  // alpha *= |S_j| (ns_engine.cpp:39)
        const uint32_t pick = ldn(nbr, at);
        bind(j, pick);
        nbound = j + 1;
#pragma unroll
        for (int q = 0; q < j; ++q)  // the pick sits at `at` in the driver: lower_bound(pick+1) = at+1
          if (q == drv) {
            hbo[q] = (uint32_t)(at - pb[q]) + 1;
            hbl[q] = pick + 1;
          }
      }
    }

    if (lane == 0) L.values[idx] = alive ? alpha : 0.0;
    if (L.bindings) {
#pragma unroll
      for (int q = 0; q < K; ++q)
        if (lane == q) L.bindings[idx * K + q] = q < nbound ? bnd[q] : INF;
    }
    if (COUNT_BYTES) bytes_acc += 32ull * __popc(used_mask);
  }
  if (COUNT_BYTES && lane == 0) atomicAdd(L.bytes_out, bytes_acc);
}

template <int K, bool CB>
void launch_k(const SampleLaunch& L, cudaStream_t s) {
  DeviceCtx& ctx = ctx_for_current_device();
  static int occ = -1;
  if (occ < 0) {
    int o = 0;
    AGPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, ns_warp_kernel<K, CB>, kThreads, 0));
    occ = o > 0 ? o : 1;
  }
  const uint64_t warps_needed = (L.count + kWarpBatch - 1) / kWarpBatch;
  uint64_t blocks = std::min<uint64_t>((uint64_t)ctx.sm_count * occ, (warps_needed + kWarps - 1) / kWarps);
  if (blocks == 0) blocks = 1;
  ns_warp_kernel<K, CB><<<(unsigned)blocks, kThreads, 0, s>>>(L);
  count_launch();
  AGPM_CUDA(cudaGetLastError());
}

}  // namespace

void launch_ns_warp(const SampleLaunch& L, cudaStream_t s) {
  const bool cb = L.bytes_out != nullptr;
#define AGPM_K(KK)              \
  case KK:                      \
    if (cb)                     \
      launch_k<KK, true>(L, s); \
    else                        \
      launch_k<KK, false>(L, s);\
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
