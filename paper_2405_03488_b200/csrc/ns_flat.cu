// Flat sampler (strategy 5): see the comment on fr_flat_kernel.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

#ifndef AGPM_FLAT_DESC_ALIGN
#define AGPM_FLAT_DESC_ALIGN 16
#endif
#define AGPM_DESC_ALIGN AGPM_FLAT_DESC_ALIGN
#ifndef AGPM_FLAT_DEDUP
#define AGPM_FLAT_DEDUP 1  // same-seed samples share the first multi-list step (see fr_flat_kernel)
#endif
#ifndef AGPM_FLAT_HINT_LOCAL_K
#define AGPM_FLAT_HINT_LOCAL_K 4
#endif
#include "frontier_common.cuh"

namespace agpm_b200 {

namespace {

// Flat sampler: one warp owns 32 samples (lane l <-> sample base + l), and
// nothing about a sample leaves the SM until its value is written.
//   * scalar work (seed, bounds, ranges, driver choice, single-list steps,
//     picks) runs lane-parallel, exactly as in fr_seed / fr_pick;
//   * a multi-list step's intersection runs over the CONCATENATION of the
//     pending samples' driver ranges, so lanes stay busy across sample
//     boundaries instead of padding every sample to whole 32-element words.
//     Fast samples (every other list a dense-core row, the driver inside the
//     core): the driver ranges are covered by aligned 32-B octets and octet o
//     of the warp's flattened cover goes to lane o % 32 (fast_round: two 16-B
//     loads, then one core-row word per element and list; the segment an octet
//     belongs to comes from a per-group bitmap of segment starts + popc and a
//     rank-indexed shared table). The rest: element e goes to lane e % 32 and
//     gets a generic per-element test;
//   * the live ballots (32 elements per word) land in shared memory; each lane
//     then counts its own segment, draws r = next_below(|S_j|) from its own
//     stream (CounterRng, or the optional Philox policy) and selects the r-th
//     live element — all lanes in parallel.
// Drivers longer than a round (kFlatW * 32 elements) take the warp-cooperative
// per-sample path (wps_sample). Bound vertices inside the
// step's [lo, hi) are failed per element (walker.hpp:70-82), so the live count
// is |S_j| directly.

constexpr int kFlatW = 64;  // ballot words per warp and round (drivers up to ~2048 elements go flat)
constexpr int kFlatThreads = 128;
constexpr int kFlatG = kFlatW / 8;  // groups (256 elements, 8 ballot words) per round

// One round of the fast class. A lane owns one OCTET of the warp's flattened
// driver range per group: eight consecutive neighbours = one aligned 32-B
// sector (two 16-B loads), then one core-row word per element and list.
// gst[g] = {bit b: a segment starts at octet R0 + 32 g + b, rank of the first
// segment starting in group g or later}; wsrc / wrows by segment rank: the byte
// address octet 0 of the flattened range would have seen from the segment, and
// the segment's two core rows. Padding slots (the neighbours of other lists
// around an unaligned driver range, or the zeroed tail of nbr[]) are probed like
// any element when they fall inside the core and skipped otherwise; their bits
// are never counted (the pick phase masks each segment to its own elements).
template <bool TWO>
__device__ __forceinline__ void fast_round(const GraphArgs& g, uint32_t R0, uint32_t Rend, int ng, const uint2* gst,
                                           const unsigned long long* wsrc, const ulonglong2* wrows, uint32_t* bal,
                                           int lane) {
  const uint32_t cb = g.core_base, wpr = g.core_wpr;
  const unsigned le_mask = (2u << lane) - 1u;
  const uint32_t o0 = R0 + lane;
#pragma unroll 1
  for (int i = 0; i < ng; ++i) {
    uint32_t bits = 0;
    const uint32_t oct = o0 + 32u * i;
    if (oct < Rend) {
      const uint2 st = gst[i];
      const uint32_t rank = (st.y + __popc(st.x & le_mask) - 1u) & 31u;
      const uint4* src = reinterpret_cast<const uint4*>(wsrc[rank] + 32ull * oct);
      const uint4 lo4 = __ldg(src), hi4 = __ldg(src + 1);
      const ulonglong2 rows = wrows[rank];
      const uint32_t* row0 = reinterpret_cast<const uint32_t*>(rows.x);
      const uint32_t* row1 = reinterpret_cast<const uint32_t*>(rows.y);
      const uint32_t a[8] = {lo4.x - cb, lo4.y - cb, lo4.z - cb, lo4.w - cb,
                             hi4.x - cb, hi4.y - cb, hi4.z - cb, hi4.w - cb};
      uint32_t m[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t w = a[k] >> 5;
        m[k] = 0;
        if (w < wpr) {
          m[k] = __ldg(row0 + w);
          if (TWO) m[k] &= __ldg(row1 + w);
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) bits |= ((m[k] >> (a[k] & 31u)) & 1u) << k;
    }
    // octet o holds elements 8 o .. 8 o + 7 of the round: word o / 4, byte o % 4
    uint32_t w = bits << ((lane & 3) * 8);
    w |= __shfl_xor_sync(FULL, w, 1);
    w |= __shfl_xor_sync(FULL, w, 2);
    if ((lane & 3) == 0) bal[8 * i + (lane >> 2)] = w;
  }
}

template <int K>
__device__ __forceinline__ bool flat_live(const GraphArgs& g, const IsectDesc<K>& d, uint32_t a) {
  const uint32_t exb = d.exb, lists = d.lists, outs = d.outs, core = d.core;
  bool fail = false;
#pragma unroll
  for (int q = 0; q < K - 1; ++q)
    if ((exb >> q) & 1u) fail = fail || a == d.owner[q];
#pragma unroll
  for (int q = 0; q < K - 1; ++q) {
    if (!((lists >> q) & 1u)) continue;
    bool found;
    if (((core >> q) & 1u) && a >= g.core_base) {
      // a lies inside the step's [lo, hi): membership in the restricted list is edge existence
      found = core_has_edge(g, d.owner[q], a);
    } else {
      const uint32_t* B = g.nbr + d.start[q];
      const uint32_t nb = d.len[q];
      const uint32_t at = lb_thread(B, 0, nb, a);
      found = at < nb && ldo(B, at) == a;
    }
    fail = fail || (found == (bool)((outs >> q) & 1u));
  }
  return !fail;
}

// bits [b0, b1) of the 32-bit word w (b0 < b1, word w overlaps the range)
__device__ __forceinline__ unsigned seg_mask(uint32_t w, uint32_t b0, uint32_t b1) {
  const uint32_t wb = w * 32;
  const uint32_t lo = b0 > wb ? b0 - wb : 0u;
  const uint32_t hi = b1 - wb >= 32 ? 32u : b1 - wb;
  const unsigned upto = hi == 32 ? FULL : (1u << hi) - 1u;
  return upto & ~((1u << lo) - 1u);
}

// A long driver, the whole warp on one sample: count the live elements, draw r
// with the sample's stream (lane src), replay the words up to the r-th. Kept
// out of line: it is rare, and inlined its registers would weigh on the hot loop.
struct WpsOut {
  unsigned long long cnt, ctr;
  uint32_t o_pick;
};

template <int K, class R>
__device__ __noinline__ WpsOut wps_sample(const GraphArgs g, const IsectDesc<K>* dp, int lane, int src, int j,
                                          R rr) {
  const IsectDesc<K>& d = *dp;
  const uint32_t core = d.core;
  const uint32_t nw = (d.dsize + 31) >> 5;
  unsigned long long c = 0;
  for (uint32_t w = 0; w < nw; ++w) c += __popc(live_word_g<K>(g, d, core, w, lane, j));
  unsigned long long r = 0;
  if (lane == src && c) r = rr.next_below(c);
  r = __shfl_sync(FULL, r, src);
  uint32_t op = 0;
  if (c) {
    for (uint32_t w = 0; w < nw; ++w) {
      const unsigned live = live_word_g<K>(g, d, core, w, lane, j);
      const unsigned pc = __popc(live);
      if (r < pc) {
        op = w * 32 + __fns(live, 0, (int)r + 1);
        break;
      }
      r -= pc;
    }
  }
  return WpsOut{c, rr.ctr, op};
}

#ifdef AGPM_FLAT_STATS
__device__ unsigned long long g_flat_stats[8];
#endif

template <int K, int kMinB, class R = CounterRng>
__global__ void __launch_bounds__(kFlatThreads, kMinB) fr_flat_kernel(const FrontierArgs A) {
  __shared__ IsectDesc<K> sdesc[kFlatThreads];
  __shared__ uint32_t sbal[kFlatThreads / 32][kFlatW];
  __shared__ uint32_t smap[kFlatThreads / 32][32];
  __shared__ unsigned long long ssrc[kFlatThreads];  // by segment rank: byte address of the segment's octet 0 - 32 * segment start
  __shared__ ulonglong2 srows[kFlatThreads];         // by segment rank: the two core rows
  __shared__ uint2 sgst[kFlatThreads / 32][kFlatG];  // by round group: {segment-start bits, rank of the first start}
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  IsectDesc<K>* wdesc = sdesc + (threadIdx.x & ~31u);
  IsectDesc<K>& my = wdesc[lane];
  uint32_t* bal = sbal[wid];
  const unsigned lt_mask = (1u << lane) - 1u;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long base = (blockIdx.x * (unsigned long long)blockDim.x) + (threadIdx.x & ~31u);
       base < A.count; base += stride) {
    const unsigned long long pos = base + lane;
    const bool act = pos < A.count;
    const unsigned long long i = act && A.order ? __ldg(A.order + pos) : pos;
    Sample<K, R> S(A.seed, A.first_id + (act ? i : 0));
    int pend = -1;
    if (act) {
      S.alpha = A.p.alpha0;
      const unsigned long long r0 = S.rng.next_below(A.g.arcs);  // ns_engine.cpp:29-33
      const unsigned long long arc = __ldg(A.g.seed_arcs + r0);
      uint32_t u = (uint32_t)(arc >> 32), v = (uint32_t)arc;
      const bool swapped = A.p.seed_ordered && u > v;
      if (swapped) {
        const uint32_t t = u;
        u = v;
        v = t;
      }
      bind(S, 0, u);
      bind(S, 1, v);
      ensure_vtx(A.g, S, 0);
      ensure_vtx(A.g, S, 1);
      if (A.g.plain) {
        if (!swapped) {
          S.hbo[0] = (uint32_t)(r0 - S.pb[0]) + 1;
          S.hbl[0] = v + 1;
        } else {
          S.hbo[1] = (uint32_t)(r0 - S.pb[1]) + 1;
          S.hbl[1] = u + 1;
          if (A.g.twin) {  // lower_bound(v1 + 1) in N(v0) through the twin arc
            S.hbo[0] = __ldg(A.g.twin + r0) + 1;
            S.hbl[0] = v + 1;
          }
        }
      }
      pend = advance<K>(A, i, S, 0, nullptr, 0, &my);
    }
    for (;;) {
      const unsigned pm = __ballot_sync(FULL, pend >= 0);
      if (!pm) break;
      __syncwarp();  // descriptors written by advance() are visible to the warp
      const int j = __shfl_sync(FULL, pend, __ffs(pm) - 1) + 2;  // every pending sample is at the same step
      const uint32_t dsz = pend >= 0 ? my.dsize : 0u;
      const bool wps = dsz > (uint32_t)kFlatW * 32 - 16;  // padded to whole octets, a fast driver still fits a round
      unsigned long long cnt = 0;
      uint32_t o_pick = 0;
#if AGPM_FLAT_DEDUP
      // Samples with the same seed pair share S_2 (the first multi-list step of a plan
      // that starts with one depends on the seed alone). In seed-sorted order they are
      // neighbours (2^24 draws over 3.1e7 arcs: 22 % of the samples repeat an arc of the
      // launch): one lane enumerates the driver, the others count and pick from its
      // ballot segment with their own streams. The key is the seed pair and which of
      // its two lists drives: equal exact ranges may resolve the driver either way
      // depending on the hints the drawn arc direction gave (ids < 2^31: the sorted
      // order is only taken up to 2^25 vertices).
      const bool dedup = j == 2 && A.order != nullptr;
      int leader = lane;
      if (dedup) {
        const unsigned long long key =
            pend >= 0 && !wps ? ((unsigned long long)(my.owner[0] | (my.drv_pos << 31)) << 32) | my.owner[1]
                              : ~(unsigned long long)lane;
        leader = __ffs(__match_any_sync(FULL, key)) - 1;
      }
      const bool follower = leader != lane;
#else
      constexpr bool dedup = false, follower = false;
      constexpr int leader = 0;
#endif
      // long drivers: the whole warp on one sample, counted, then replayed up to
      // the r-th live element
      for (unsigned bm = __ballot_sync(FULL, wps); bm; bm &= bm - 1) {
        const int src = __ffs(bm) - 1;
        const WpsOut o = wps_sample<K>(A.g, wdesc + src, lane, src, j, S.rng);
        if (lane == src) {
          cnt = o.cnt;
          o_pick = o.o_pick;
          S.rng.ctr = o.ctr;
        }
      }
      // fast path (the common case on a relabelled graph): every other list is a
      // core row, the driver lies in the core, no out-lists and no bound vertex
      // inside [lo, hi) -> per element one driver load and one bit per list
      const uint32_t cb = A.g.core_base;
      bool fast = false;
      if (pend >= 0 && !wps) {
        const uint32_t l = my.lists;
        // a bound vertex inside [lo, hi) that owns one of this step's lists cannot be a
        // candidate on a loop-free view (it is not in its own list): only the others count
        // (the 4-cycle's S_3 = N(v0) & N(v2) above v1, where v2 itself may exceed v1)
        const uint32_t own = l | (my.drv_pos < 32 ? 1u << my.drv_pos : 0u);
        const uint32_t exb = A.g.loop_free ? my.exb & ~own : my.exb;
        fast = my.core == (l | (1u << 31)) && my.outs == 0 && exb == 0 && __popc(l) <= 2;
#ifdef AGPM_FLAT_STATS
        const uint32_t exe = my.exb & ~(l | (my.drv_pos < 31 ? 1u << my.drv_pos : 0u));
        const bool allcore = (my.core & 0x7fffffffu) == l && my.outs == 0 && __popc(l) <= 2;
        atomicAdd(&g_flat_stats[0], 1ull);
        atomicAdd(&g_flat_stats[1], (unsigned long long)fast);
        atomicAdd(&g_flat_stats[2], (unsigned long long)(allcore && (my.core >> 31) && exe == 0));
        atomicAdd(&g_flat_stats[3], (unsigned long long)(allcore && exe == 0));
        atomicAdd(&g_flat_stats[4], (unsigned long long)dsz);
        if (fast) atomicAdd(&g_flat_stats[5], (unsigned long long)dsz);
        if (allcore && exe == 0) atomicAdd(&g_flat_stats[6], (unsigned long long)dsz);
#endif
      }
#ifdef AGPM_FLAT_STATS
      if (wps) atomicAdd(&g_flat_stats[7], 1ull);
#endif
      // the rest: flattened element-parallel rounds of <= kFlatW * 32 elements,
      // fast samples first, then the others (each class flattened on its own)
      for (int cls = 0; cls < 2; ++cls) {
      const bool allfast = cls == 0;
      const bool part = pend >= 0 && !wps && fast == allfast && !follower;
      // fast class: units are octets of the 32-B-aligned cover of the driver range
      const uint32_t head = (uint32_t)(reinterpret_cast<unsigned long long>(my.drv) >> 2) & 7u;
      const uint32_t sz = !part ? 0u : allfast ? (head + dsz + 7) >> 3 : dsz;
      const uint32_t round_units = allfast ? (uint32_t)kFlatW * 4 : (uint32_t)kFlatW * 32;
      uint32_t P = sz;  // inclusive prefix of segment sizes over lanes
#pragma unroll
      for (int dd = 1; dd < 32; dd <<= 1) {
        const uint32_t t = __shfl_up_sync(FULL, P, dd);
        if (lane >= dd) P += t;
      }
      const uint32_t excl = P - sz;
      const uint32_t total = __shfl_sync(FULL, P, 31);
      if (total == 0) continue;
      const unsigned partm = __ballot_sync(FULL, part);
      __syncwarp();
      if (part) {
        const uint32_t rank = __popc(partm & lt_mask);
        smap[wid][rank] = (uint32_t)lane;
        if (allfast) {  // the fast table is indexed by segment rank: no lane lookup in the loop
          const uint32_t l = my.lists;
          const int q0 = __ffs(l) - 1, q1 = 31 - __clz(l);
          ssrc[(threadIdx.x & ~31u) + rank] =
              (reinterpret_cast<unsigned long long>(my.drv) & ~31ull) - 32ull * excl;
          srows[(threadIdx.x & ~31u) + rank] = make_ulonglong2(
              reinterpret_cast<unsigned long long>(A.g.core + (unsigned long long)(my.owner[q0] - cb) * A.g.core_wpr),
              reinterpret_cast<unsigned long long>(A.g.core + (unsigned long long)(my.owner[q1] - cb) * A.g.core_wpr));
        }
      }
      __syncwarp();
      const uint32_t lane_of_rank = smap[wid][lane];
      const unsigned long long* wsrc = ssrc + (threadIdx.x & ~31u);
      const ulonglong2* wrows = srows + (threadIdx.x & ~31u);
      uint2* gst = sgst[wid];
      // one or two other lists: the same for every fast sample of the warp (same step, driver among the in-lists)
      const bool two = __any_sync(FULL, part && allfast && __popc(my.lists) == 2);
      for (uint32_t R0 = 0; R0 < total;) {
        const uint32_t Rend = __reduce_max_sync(FULL, P <= R0 + round_units ? P : 0u);
        uint32_t rk = __popc(__ballot_sync(FULL, part && P <= R0));  // segments of earlier rounds
        uint32_t it = 0;
        const bool inr = part && excl >= R0 && P <= Rend;  // this lane's segment is in the round
        uint32_t b0 = excl - R0, b1 = P - R0;               // its bits in bal[]
        if (allfast) {
          const int ng = (int)((Rend - R0 + 31) >> 5);
          if (lane < kFlatG) gst[lane].x = 0;
          __syncwarp();
          if (inr) atomicOr(&gst[(excl - R0) >> 5].x, 1u << ((excl - R0) & 31));
          __syncwarp();
          {
            const uint32_t c0 = lane < kFlatG ? __popc(gst[lane].x) : 0u;
            uint32_t s0 = c0;
#pragma unroll
            for (int dd = 1; dd < kFlatG; dd <<= 1) {
              const uint32_t t0 = __shfl_up_sync(FULL, s0, dd);
              if (lane >= dd) s0 += t0;
            }
            if (lane < kFlatG) gst[lane].y = rk + s0 - c0;
          }
          __syncwarp();
          if (two)
            fast_round<true>(A.g, R0, Rend, ng, gst, wsrc, wrows, bal, lane);
          else
            fast_round<false>(A.g, R0, Rend, ng, gst, wsrc, wrows, bal, lane);
          b0 = b0 * 8 + head;
          b1 = b0 + dsz;
        } else
        for (uint32_t e0 = R0; e0 < Rend; e0 += 32, ++it) {
          const unsigned starts =
              __reduce_or_sync(FULL, (part && excl >= e0 && excl < e0 + 32) ? 1u << (excl - e0) : 0u);
          const uint32_t rank = rk + __popc(starts & ((2u << lane) - 1u)) - 1u;
          rk += __popc(starts);
          const uint32_t e = e0 + lane;
          const int src = (int)__shfl_sync(FULL, lane_of_rank, (int)(rank & 31u));
          const uint32_t ex_src = __shfl_sync(FULL, excl, src);
          bool live = false;
          if (e < Rend) {
            const IsectDesc<K>& d = wdesc[src];
            live = flat_live<K>(A.g, d, ldo(d.drv, e - ex_src));
          }
          const unsigned b = __ballot_sync(FULL, live);
          if (lane == 0) bal[it] = b;
        }
        __syncwarp();
        bool mine = inr;
        if (dedup) {  // a follower reads its leader's segment
          const bool l_inr = __shfl_sync(FULL, inr, leader);
          const uint32_t lb0 = __shfl_sync(FULL, b0, leader), lb1 = __shfl_sync(FULL, b1, leader);
          if (follower && l_inr && fast == allfast) {
            mine = true;
            b0 = lb0;
            b1 = lb1;
          }
        }
        if (mine) {
          const uint32_t w0 = b0 >> 5, w1 = (b1 - 1) >> 5;
          unsigned long long c = 0;
          for (uint32_t w = w0; w <= w1; ++w) c += __popc(bal[w] & seg_mask(w, b0, b1));
          cnt = c;
          if (c) {
            unsigned long long r = S.rng.next_below(c);
            for (uint32_t w = w0; w <= w1; ++w) {
              const unsigned m = bal[w] & seg_mask(w, b0, b1);
              const unsigned pc = __popc(m);
              if (r < pc) {
                o_pick = w * 32 + __fns(m, 0, (int)r + 1) - b0;
                break;
              }
              r -= pc;
            }
          }
        }
        __syncwarp();
        R0 = Rend;
      }
      }
      if (pend >= 0) {
        if (cnt == 0) {
          finish(A, i, S, j, false);
          pend = -1;
        } else {
          S.alpha = __dmul_rn(S.alpha, (double)cnt);  // alpha *= |S_j| (ns_engine.cpp:39)
          const uint32_t pick = ldo(my.drv, o_pick);
          const uint32_t dpos = my.drv_pos, drs = my.drv_rs;
          if (dpos != NO_DRV) {
#pragma unroll
            for (int q = 0; q < K; ++q)
              if ((uint32_t)q == dpos) {  // lower_bound(pick + 1) = drv_rs + o + 1
                S.hbo[q] = drs + o_pick + 1;
                S.hbl[q] = pick + 1;
              }
          }
          uint32_t from = 0;
#pragma unroll
          for (int q = 0; q < K; ++q)
            if ((uint32_t)q == dpos) from = S.bnd[q];
          bind(S, j, pick);
          if (A.p.twin_hint[pend] && A.g.twin && dpos != NO_DRV) {  // position of v_drv in N(pick)
            const uint32_t tw = __ldg(A.g.twin + (unsigned long long)(my.drv - A.g.nbr) + o_pick) + 1;
            // Placement: for K >= 4 the hint arrays are addressed with the runtime
            // position j here, which puts them in local memory (an L1-resident
            // stack) instead of competing for the 48 registers of the hot loop —
            // measured per 2^24 samples: 4-clique 8.15 -> 7.75 ms, 5-clique 11.8 ->
            // 10.6 ms; K = 3 keeps them in registers (triangle 5.13 vs 5.38 ms).
            if constexpr (K >= AGPM_FLAT_HINT_LOCAL_K) {
              S.hbo[j] = tw;
              S.hbl[j] = from + 1;
            } else {
#pragma unroll
              for (int q = 2; q < K; ++q)
                if (q == j) {
                  S.hbo[q] = tw;
                  S.hbl[q] = from + 1;
                }
            }
          }
          pend = advance<K>(A, i, S, pend + 1, nullptr, 0, &my);
        }
      }
    }
  }
}

// Processing order. Sample ids are independent streams and values / bindings are
// written by id, so the order in which a launch works through its ids is free.
// In seed-sorted order consecutive samples (the 32 lanes of a warp, the warps of
// a block) share their hub and mostly their seed edge's neighbourhood: vertex
// records, adjacency lists and dense-core rows are then read through L1 / L2
// instead of DRAM. A pre-pass draws every id's seed (the draw the sampler
// repeats) and a radix sort of (key, id) pairs orders the ids, ~0.3 ms per 2^24.
// Two keys:
//   * the seed arc's index (arc order = source vertex, then target): no gather in
//     the pre-pass and coalesced seed-arc gathers in the sampler — plans with two
//     multi-list steps (4-clique), and every plan above 2^22 vertices;
//   * composite: the top 16 bits of the smaller seed endpoint, then the top 16 of the
//     larger (neighbouring seed EDGES whichever arc was drawn) — deeper plans up to
//     2^22 vertices.
// Taken where it pays: launches of >= 2^20 ids; plans with at least two multi-list
// steps on graphs up to 2^25 vertices, plans with one up to 2^21. Per 2^24 samples,
// sort included, id order -> sorted (with the shared first step, see the kernel):
//   arc key, 4-clique: RMAT-20 5.91 -> 5.03 ms, RMAT-21 7.15 -> 6.30, RMAT-22 8.55 -> 7.66,
//     RMAT-23 10.24 -> 9.53, RMAT-24 12.76 -> 11.96, RMAT-25 16.17 -> 15.43 (the top 24 key
//     bits: three sort passes; all 25 bits, four passes: RMAT-20 5.15; 16 bits: 5.38);
//   composite key: RMAT-20 5-clique 9.64 -> 7.97, 6-clique 15.7 -> 12.9, RMAT-22 5-clique
//     12.0 -> 11.7; beyond it loses (RMAT-23 5-clique 14.57 -> 14.67, RMAT-24 16.9 -> 17.8)
//     where the arc key still wins (5-clique RMAT-23 14.53 -> 13.53, RMAT-24 17.06 -> 16.04,
//     RMAT-25 21.19 -> 20.12; 6-clique RMAT-24 24.3 -> 22.6);
//     on the RMAT-20 4-clique: 5.57 (arc key 5.31, before the shared step); the smaller
//     endpoint alone 5.70 / 5-clique 8.26, the larger alone 5.70 / 8.84, 12 or 8 bits
//     5.99 / 8.61 and 5.87 / 8.56.
//   arc key, one multi-list step: RMAT-20 triangle 3.19 -> 2.92, 4-cycle 5.12 -> 4.67; not
//     beyond 2^21 vertices (RMAT-22 triangle 5.20 -> 5.20, 4-cycle 7.15 -> 7.30; with the
//     composite key RMAT-20 triangle 3.16 -> 3.45, RMAT-22 4-cycle 7.06 -> 7.74);
//   RMAT-26 4-clique (512 K core): 22.4 -> 22.6, not taken.
#ifndef AGPM_FLAT_ARC_BITS
#define AGPM_FLAT_ARC_BITS 24
#endif
#ifndef AGPM_FLAT_SORT
#define AGPM_FLAT_SORT 1  // 0: always id order
#endif
template <class R>
__global__ void flat_seedkey_kernel(GraphArgs g, unsigned long long seed, unsigned long long first_id,
                                    unsigned long long count, bool arc_key, int shift,
                                    uint32_t* __restrict__ keys, uint32_t* __restrict__ idx) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < count;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    R rng(seed, 0, first_id + i);
    const unsigned long long r0 = rng.next_below(g.arcs);  // ns_engine.cpp:29-33
    uint32_t key;
    if (arc_key) {
      key = (uint32_t)(r0 >> shift);
    } else {
      const unsigned long long arc = __ldg(g.seed_arcs + r0);
      const uint32_t u = (uint32_t)(arc >> 32), v = (uint32_t)arc;
      key = ((min(u, v) >> shift) << 16) | (max(u, v) >> shift);
    }
    keys[i] = key;
    idx[i] = (uint32_t)i;
  }
}

template <class R>
const uint32_t* flat_order(const SampleLaunch& L, int multi_steps, cudaStream_t s) {
  // (16 B of sort scratch per id: launches beyond 2^26 ids — the library's own drivers
  // launch at most 2^24 at a time — keep id order)
  const bool arc_key = multi_steps <= 2 || L.g.n > (1u << 22);
  if (!AGPM_FLAT_SORT || multi_steps < 1 || L.g.n > (multi_steps == 1 ? 1u << 21 : 1u << 25) ||
      L.count < (1ull << 20) ||
      L.count > (1ull << 26))
    return nullptr;
  DeviceCtx& ctx = ctx_for_current_device();
  const size_t n = (size_t)L.count;
  auto* buf = static_cast<uint32_t*>(ctx.get(12, 16 * n));  // keys in/out, ids in/out
  uint32_t *k0 = buf, *k1 = buf + n, *i0 = buf + 2 * n, *i1 = buf + 3 * n;
  auto bits_of = [](unsigned long long x) {
    int b = 1;
    while (b < 63 && (1ull << b) < x) ++b;
    return b;
  };
  // keys: the top AGPM_FLAT_ARC_BITS bits of the arc index (three 8-bit sort passes), or
  // 16 + 16 top bits of the endpoints (four)
  const int width = arc_key ? bits_of(L.g.arcs) : bits_of(L.g.n);
  const int shift = std::max(0, width - (arc_key ? AGPM_FLAT_ARC_BITS : 16));
  const int end_bit = arc_key ? width - shift : 2 * 16;
  flat_seedkey_kernel<R><<<(unsigned)std::min<size_t>((n + 255) / 256, (size_t)ctx.sm_count * 16), 256, 0, s>>>(
      L.g, L.seed, L.first_id, L.count, arc_key, shift, k0, i0);
  count_launch();
  size_t temp = 0;
  AGPM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, k0, k1, i0, i1, n, 0, end_bit, s));
  void* tmp = ctx.get(13, temp);
  AGPM_CUDA(cub::DeviceRadixSort::SortPairs(tmp, temp, k0, k1, i0, i1, n, 0, end_bit, s));
  count_launch(1 + (end_bit + 7) / 8);  // histogram + one onesweep pass per 8 key bits
  return i1;
}

template <int K, class R>
void run_flat_k(const SampleLaunch& L, cudaStream_t s) {
  DeviceCtx& ctx = ctx_for_current_device();
  FrontierArgs A{};
  A.g = L.g;
  A.p = L.p;
  A.seed = L.seed;
  A.first_id = L.first_id;
  A.count = L.count;
  A.values = L.values;
  A.bindings = L.bindings;
  int multi_steps = 0;
  for (int st = 0; st < K - 2; ++st) {
    const unsigned in_m = L.p.in_mask[st], out_m = L.p.out_mask[st];
    A.step_multi[st] = !(__builtin_popcount(in_m) == 1 && out_m == 0);
    A.step_reuse[st] = 0;
    multi_steps += A.step_multi[st];
  }
  A.order = flat_order<R>(L, multi_steps, s);
  // Resident 128-thread blocks per SM (the register cap): the kernel hides latency with
  // warps, but shared memory and local-memory stack compete with L1 for the same 256 KB,
  // so 8 blocks (64 registers, no spills, 19 KB of tables each) beat 9 and 10.
  // Measured per 2^24 samples on the config-2 graph (triangle / 4-clique / 5-clique):
  // 7 blocks 3.35 / 6.05 / 9.99 ms, 8 blocks 3.15 / 5.83 / 9.47, 9 blocks 3.15 / 5.91 / 9.78,
  // 10 blocks (48 registers, spills) 3.28 / 6.23 / 12.9.
#ifndef AGPM_FLAT_MINB45
#define AGPM_FLAT_MINB45 8
#endif
  constexpr int kMinB = K <= 5 ? AGPM_FLAT_MINB45 : 8;
  auto kern = fr_flat_kernel<K, kMinB, R>;
  static int occ = -1;
  if (occ < 0) {
#ifdef AGPM_FLAT_CARVEOUT
    AGPM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, AGPM_FLAT_CARVEOUT));
#endif
    int o = 0;
    AGPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, kFlatThreads, 0));
    occ = std::max(o, 1);
  }
  // AGPM_FLAT_WAVES > 0: at most that many resident waves of blocks (a grid-
  // stride loop); 0: one block per 128 samples, so blocks retire continuously
  // and kernels of other streams (a view being uploaded and indexed on another
  // host thread) are scheduled in between instead of waiting for the launch
#ifndef AGPM_FLAT_WAVES
#define AGPM_FLAT_WAVES 1
#endif
  const unsigned long long want = (L.count + kFlatThreads - 1) / kFlatThreads;
  const unsigned long long cap =
      AGPM_FLAT_WAVES > 0 ? (unsigned long long)ctx.sm_count * occ * AGPM_FLAT_WAVES : want;
  const unsigned blocks = (unsigned)std::max<unsigned long long>(1, std::min<unsigned long long>(want, cap));
  kern<<<blocks, kFlatThreads, 0, s>>>(A);
  count_launch();
  AGPM_CUDA(cudaGetLastError());
#ifdef AGPM_FLAT_STATS
  {
    unsigned long long h[8], z[8] = {};
    cudaStreamSynchronize(s);
    cudaMemcpyFromSymbol(h, g_flat_stats, sizeof(h));
    cudaMemcpyToSymbol(g_flat_stats, z, sizeof(z));
    fprintf(stderr, "flat stats: multi-steps %llu fast %llu fast+exb_eff %llu allcore(any lo) %llu | elements %llu fast %llu allcore %llu | wps %llu\n",
            h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
  }
#endif
}

}  // namespace

void launch_ns_flat(const SampleLaunch& L, cudaStream_t s, bool philox) {
  if (L.bytes_out) throw std::invalid_argument("B_min accounting runs on the warp sampler");
  switch (L.p.k) {
    case 3: philox ? run_flat_k<3, PhiloxRng>(L, s) : run_flat_k<3, CounterRng>(L, s); break;
    case 4: philox ? run_flat_k<4, PhiloxRng>(L, s) : run_flat_k<4, CounterRng>(L, s); break;
    case 5: philox ? run_flat_k<5, PhiloxRng>(L, s) : run_flat_k<5, CounterRng>(L, s); break;
    case 6: philox ? run_flat_k<6, PhiloxRng>(L, s) : run_flat_k<6, CounterRng>(L, s); break;
    case 7: philox ? run_flat_k<7, PhiloxRng>(L, s) : run_flat_k<7, CounterRng>(L, s); break;
    case 8: philox ? run_flat_k<8, PhiloxRng>(L, s) : run_flat_k<8, CounterRng>(L, s); break;
    case 9: philox ? run_flat_k<9, PhiloxRng>(L, s) : run_flat_k<9, CounterRng>(L, s); break;
    default: throw std::invalid_argument("device sampler needs 3 <= k <= 9");
  }
}

}  // namespace agpm_b200
