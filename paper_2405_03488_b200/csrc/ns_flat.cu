// Flat sampler (strategy 5): see the comment on fr_flat_kernel.
#include <algorithm>
#include <cstdlib>
#include <stdexcept>

#ifndef AGPM_FLAT_DESC_ALIGN
#define AGPM_FLAT_DESC_ALIGN 16
#endif
#define AGPM_DESC_ALIGN AGPM_FLAT_DESC_ALIGN
#include "frontier_common.cuh"

namespace agpm_b200 {

namespace {

// Flat sampler: one warp owns 32 samples (lane l <-> sample base + l), and
// nothing about a sample leaves the SM until its value is written.
//   * scalar work (seed, bounds, ranges, driver choice, single-list steps,
//     picks) runs lane-parallel, exactly as in fr_seed / fr_pick;
//   * a multi-list step's intersection runs over the CONCATENATION of the
//     pending samples' driver ranges: element e of the warp's flattened range
//     goes to lane e % 32, whose segment rank is found from a reduction of
//     the segment starts (one redux + popc; the fast class reads its driver
//     and core rows from a rank-indexed shared table), so lanes stay busy
//     across sample boundaries instead of padding every sample to whole
//     32-element words; fast samples (every other list a dense-core row, the
//     driver inside the core) cost one driver load and one bit per list per
//     element, the rest a generic per-element test;
//   * the live ballots (32 elements per word) land in shared memory; each lane
//     then counts its own segment, draws r = next_below(|S_j|) from its own
//     stream (CounterRng, or the optional Philox policy) and selects the r-th
//     live element — all lanes in parallel.
// Drivers longer than kFlatW * 32 elements take the warp-cooperative
// per-sample path of the fused kernel (live_word). Bound vertices inside the
// step's [lo, hi) are failed per element (walker.hpp:70-82), so the live count
// is |S_j| directly.
constexpr int kFlatW = 64;  // ballot words per warp and round (drivers up to 2048 elements go flat)
constexpr int kFlatThreads = 128;
#ifndef AGPM_FLAT_U
#define AGPM_FLAT_U 2  // driver words in flight per warp in the fast loop
#endif

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

template <int K, int kFlatU, int kMinB, class R = CounterRng>
__global__ void __launch_bounds__(kFlatThreads, kMinB) fr_flat_kernel(const FrontierArgs A) {
  __shared__ IsectDesc<K> sdesc[kFlatThreads];
  __shared__ uint32_t sbal[kFlatThreads / 32][kFlatW];
  __shared__ uint32_t smap[kFlatThreads / 32][32];
  __shared__ uint4 sfast[kFlatThreads];
  __shared__ uint32_t sexcl[kFlatThreads];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  IsectDesc<K>* wdesc = sdesc + (threadIdx.x & ~31u);
  IsectDesc<K>& my = wdesc[lane];
  uint32_t* bal = sbal[wid];
  const unsigned lt_mask = (1u << lane) - 1u;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long base = (blockIdx.x * (unsigned long long)blockDim.x) + (threadIdx.x & ~31u);
       base < A.count; base += stride) {
    const unsigned long long i = base + lane;
    const bool act = i < A.count;
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
      const bool wps = dsz > (uint32_t)kFlatW * 32;
      unsigned long long cnt = 0;
      uint32_t o_pick = 0;
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
        fast = my.core == (l | (1u << 31)) && my.outs == 0 && my.exb == 0 && __popc(l) <= 2;
      }
      // the rest: flattened element-parallel rounds of <= kFlatW * 32 elements,
      // fast samples first, then the others (each class flattened on its own)
      for (int cls = 0; cls < 2; ++cls) {
      const bool allfast = cls == 0;
      const bool part = pend >= 0 && !wps && fast == allfast;
      const uint32_t sz = part ? dsz : 0u;
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
          const unsigned long long dp = reinterpret_cast<unsigned long long>(my.drv);
          sfast[(threadIdx.x & ~31u) + rank] = make_uint4((uint32_t)dp, (uint32_t)(dp >> 32),
                                                          (my.owner[q0] - cb) * A.g.core_wpr,
                                                          (my.owner[q1] - cb) * A.g.core_wpr);
          sexcl[(threadIdx.x & ~31u) + rank] = excl;
        }
      }
      __syncwarp();
      const uint32_t lane_of_rank = smap[wid][lane];
      const uint4* wfast = sfast + (threadIdx.x & ~31u);
      const uint32_t* wexcl = sexcl + (threadIdx.x & ~31u);
      for (uint32_t R0 = 0; R0 < total;) {
        const uint32_t Rend = __reduce_max_sync(FULL, P <= R0 + (uint32_t)kFlatW * 32 ? P : 0u);
        uint32_t rk = __popc(__ballot_sync(FULL, part && P <= R0));  // segments of earlier rounds
        uint32_t it = 0;
        if (allfast) {
          // kFlatU independent words in flight per warp: their driver loads, then their bit probes
          for (uint32_t e0 = R0; e0 < Rend; e0 += 32 * kFlatU, it += kFlatU) {
            uint32_t a[kFlatU], rw0[kFlatU], rw1[kFlatU];
            bool v[kFlatU];
#pragma unroll
            for (int u = 0; u < kFlatU; ++u) {
              const uint32_t eb = e0 + 32 * u;
              const unsigned starts =
                  __reduce_or_sync(FULL, (part && excl >= eb && excl < eb + 32) ? 1u << (excl - eb) : 0u);
              const uint32_t rank = rk + __popc(starts & ((2u << lane) - 1u)) - 1u;
              rk += __popc(starts);
              const uint4 f = wfast[rank & 31u];
              const uint32_t ex_src = wexcl[rank & 31u];
              v[u] = eb + lane < Rend;
              const uint32_t* drv = reinterpret_cast<const uint32_t*>(((unsigned long long)f.y << 32) | f.x);
              a[u] = v[u] ? ldo(drv, eb + lane - ex_src) - cb : 0u;
              rw0[u] = f.z;
              rw1[u] = f.w;
            }
#pragma unroll
            for (int u = 0; u < kFlatU; ++u) {
              bool live = false;
              if (v[u]) {
                const uint32_t c = a[u];
                const uint32_t b0 = __ldg(A.g.core + rw0[u] + (c >> 5));
                const uint32_t b1 = __ldg(A.g.core + rw1[u] + (c >> 5));
                live = ((b0 & b1) >> (c & 31)) & 1u;
              }
              const unsigned b = __ballot_sync(FULL, live);
              if (lane == 0) bal[it + u] = b;
            }
          }
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
        if (part && excl >= R0 && P <= Rend) {  // this lane's segment is in the round
          const uint32_t b0 = excl - R0, b1 = P - R0;
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
            if constexpr (K >= 4) {
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
  for (int st = 0; st < K - 2; ++st) {
    const unsigned in_m = L.p.in_mask[st], out_m = L.p.out_mask[st];
    A.step_multi[st] = !(__builtin_popcount(in_m) == 1 && out_m == 0);
    A.step_reuse[st] = 0;
  }
  // 2 words in flight per warp; registers capped by the resident 128-thread
  // blocks per SM: the loop is latency bound, so occupancy beats the few spills
  // a cap costs. Measured per 2^24 samples on the config-2 graph: 4-clique 96
  // regs 14.2 ms, 64 regs 9.1, 56 regs 8.9, 48 regs 8.8, 40 regs 9.9; triangle
  // 64 regs 5.5 vs 48 regs 5.8; 5-clique 48 regs 12.3 vs 64 regs 13.4.
#ifndef AGPM_FLAT_MINB45
#define AGPM_FLAT_MINB45 10
#endif
  constexpr int kMinB = K == 3 ? 8 : K <= 5 ? AGPM_FLAT_MINB45 : 8;
  auto kern = fr_flat_kernel<K, AGPM_FLAT_U, kMinB, R>;
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
