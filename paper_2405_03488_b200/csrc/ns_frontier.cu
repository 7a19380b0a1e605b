// Frontier (phase) sampler: the throughput strategy for large batches.
//
// A batch of samples advances through the plan one multi-list step at a time:
//
//   advance  (1 thread / sample)   seed draw; bound-restricted ranges of the
//            step's lists (per-thread lower_bound narrowed by hints: vtx.up,
//            the seed arc index, the previous pick's index); single-list steps
//            resolved inline by index arithmetic; driver = smallest range;
//            writes an IsectDesc and the sample's bitmap word count.
//   scan     (CUB)                  word offsets: every sample's hit bitmap
//            starts on a 32-bit word boundary.
//   isect    (1 warp / bitmap word) a word = 32 driver elements of ONE sample.
//            A test "a in list q" is one bit of the dense-core matrix when q's
//            owner is a core vertex (the driver already sits inside the step's
//            [lo, hi), so membership is edge existence); otherwise the warp
//            loads 32 splitters of list q, finds each lane's bucket with a
//            5-step shuffle search and finishes with a short per-lane search.
//            One ballot -> the fail word. No atomics, no memset.
//   pick     (1 thread / sample)    |S_j| = |D| - fails - bound vertices,
//            r = next_below(|S_j|), r-th surviving bit -> v_j, alpha *= |S_j|.
//            Nested reuse: when step j+1's lists contain step j's (cliques),
//            S_{j+1} = {x in S_j : x in [lo', hi'), x != v_j} ∩ (new lists) —
//            the survivors are compacted (warp-aggregated allocation) and become
//            the next driver, so step j+1 intersects a handful of elements
//            with ONE new list instead of re-intersecting all of them.
//
// Candidate sets and picks are exactly build_step_candidates +
// cand[next_below(|cand|)] (walker.hpp:30-83, ns_engine.cpp:27-53) with the
// sample's own CounterRng(seed, 0, id): the set S_j does not depend on how it
// is computed, so results are bit-identical to the warp/lane kernels and to the
// reference's draw_sample with workers = 1.
#include <cub/cub.cuh>

#include <algorithm>
#include <stdexcept>

#include "frontier_common.cuh"
#ifndef AGPM_ISECT_QUAD
#define AGPM_ISECT_QUAD 1  // ... and four at a time before that (12.86 -> 12.41 ms)
#endif
#ifndef AGPM_ISECT_PAIR
#define AGPM_ISECT_PAIR 1  // fast path two words at a time (RMAT-22 4-cycle 13.32 -> 12.86 ms per 2^24)
#endif
#ifndef AGPM_TWIN_HINT_MULTI
#define AGPM_TWIN_HINT_MULTI 0  // see AGPM_TWIN_HINT_SINGLE
#endif

namespace agpm_b200 {

namespace {

template <int K>
__global__ void __launch_bounds__(256) fr_seed_kernel(const FrontierArgs A) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < A.count;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    Sample<K> S(A.seed, A.first_id + i);
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
    if (A.g.plain) {  // arc r0 is nbr[r0] in its source's list
      // and, with twin arcs, its source sits at twin[r0] in the target's list
      const uint32_t tw = A.g.twin ? __ldg(A.g.twin + r0) + 1 : 0u;
      if (!swapped) {
        S.hbo[0] = (uint32_t)(r0 - S.pb[0]) + 1;
        S.hbl[0] = v + 1;
        if (tw) {  // lower_bound(v0 + 1) in N(v1)
          S.hbo[1] = tw;
          S.hbl[1] = u + 1;
        }
      } else {
        S.hbo[1] = (uint32_t)(r0 - S.pb[1]) + 1;
        S.hbl[1] = u + 1;
        if (tw) {  // lower_bound(v1 + 1) in N(v0)
          S.hbo[0] = tw;
          S.hbl[0] = v + 1;
        }
      }
    }
    advance<K>(A, i, S, 0, nullptr, 0);
  }
}

// One warp per bitmap word; each warp walks a contiguous run of words. The run
// is consumed sample by sample: the owning sample is located once (k-ary over
// the word offsets, then 32 offsets per probe), its descriptor is read once
// into registers, and its words follow. Core lists cost one L2 word per lane;
// the rest load 32 splitters and finish with a short per-lane search.
template <int K>
__global__ void __launch_bounds__(256, 8) fr_isect_kernel(const FrontierArgs A, unsigned long long words) {
  const int lane = threadIdx.x & 31;
  const unsigned long long* __restrict__ off = A.offsets;
  const IsectDesc<K>* __restrict__ desc = reinterpret_cast<const IsectDesc<K>*>(A.desc);
  const uint32_t* __restrict__ nbr = A.g.nbr;
  const unsigned long long warp = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
  const unsigned long long nwarps = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
  const unsigned long long per = (words + nwarps - 1) / nwarps;
  const unsigned long long w0 = warp * per, w1 = min(words, w0 + per);
  if (w0 >= w1) return;
  unsigned long long s;
  {  // last s with off[s] <= w0
    unsigned long long lo = 0, hi = A.count;
    while (hi - lo > 32) {
      const unsigned long long step = (hi - lo) / 33;
      const unsigned c = __popc(__ballot_sync(FULL, off[lo + (unsigned long long)(lane + 1) * step] <= w0));
      const unsigned long long nlo = c ? lo + c * step : lo;
      hi = c < 32 ? lo + (c + 1) * step : hi;
      lo = nlo;
    }
    const unsigned long long pos = lo + lane;
    s = lo + __popc(__ballot_sync(FULL, pos < hi && off[pos] <= w0)) - 1;
  }
  unsigned long long w = w0;
  while (w < w1) {
    // s = last sample with off[s] <= w (offsets are non-decreasing: a prefix test)
    for (;;) {
      const unsigned long long t = s + 1 + lane;
      const unsigned m = __ballot_sync(FULL, t <= A.count && off[t] <= w);
      s += __popc(m);
      if (m != FULL) break;
    }
    const unsigned long long we = min(w1, off[s + 1]);
    const IsectDesc<K>& d = desc[s];
    // loop-invariant scalars of the descriptor in registers; per-list fields stay in L1
    const uint32_t* __restrict__ drv = d.drv;
    const uint32_t dsize = d.dsize, lists = d.lists, outs = d.outs, core0 = d.core;
    const unsigned long long wbase = off[s];
    if (core0 == (lists | (1u << 31)) && outs == 0 && __popc(lists) <= 2) {
      // fast path (the common case on a relabelled graph): every other list is
      // a core row and the whole driver lies inside the core -> per word one
      // coalesced driver load and one bit probe per list
      const int q0 = __ffs(lists) - 1;
      const int q1 = __popc(lists) == 2 ? 31 - __clz(lists) : -1;
      const uint32_t cb = A.g.core_base;
      const uint32_t* r0 = A.g.core + (unsigned long long)(d.owner[q0] - cb) * A.g.core_wpr;
      const uint32_t* r1 = q1 >= 0 ? A.g.core + (unsigned long long)(d.owner[q1] - cb) * A.g.core_wpr : r0;
#if AGPM_ISECT_QUAD
      for (; w + 3 < we; w += 4) {  // four words: the driver loads, then the probes
        const uint32_t o = (uint32_t)(w - wbase) * 32 + lane;
        uint32_t c[4], a[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) c[u] = o + 32 * u < dsize ? ldo(drv, o + 32 * u) - cb : 0u;
#pragma unroll
        for (int u = 0; u < 4; ++u) a[u] = __ldg(r0 + (c[u] >> 5)) & __ldg(r1 + (c[u] >> 5));
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const unsigned bal = __ballot_sync(FULL, o + 32 * u < dsize && !((a[u] >> (c[u] & 31)) & 1u));
          if (lane == 0) A.bitmap[w + u] = bal;
        }
      }
#endif
#if AGPM_ISECT_PAIR
      // two words per iteration: both driver loads, then the four bit probes
      for (; w + 1 < we; w += 2) {
        const uint32_t o = (uint32_t)(w - wbase) * 32 + lane;
        const bool v0 = o < dsize, v1 = o + 32 < dsize;
        const uint32_t c0 = v0 ? ldo(drv, o) - cb : 0u;
        const uint32_t c1 = v1 ? ldo(drv, o + 32) - cb : 0u;
        const uint32_t a0 = __ldg(r0 + (c0 >> 5)) & __ldg(r1 + (c0 >> 5));
        const uint32_t a1 = __ldg(r0 + (c1 >> 5)) & __ldg(r1 + (c1 >> 5));
        const unsigned bal0 = __ballot_sync(FULL, v0 && !((a0 >> (c0 & 31)) & 1u));
        const unsigned bal1 = __ballot_sync(FULL, v1 && !((a1 >> (c1 & 31)) & 1u));
        if (lane == 0) {
          A.bitmap[w] = bal0;
          A.bitmap[w + 1] = bal1;
        }
      }
#endif
      for (; w < we; ++w) {
        const uint32_t o = (uint32_t)(w - wbase) * 32 + lane;
        bool fail = false;
        if (o < dsize) {
          const uint32_t c = ldo(drv, o) - cb;
          const uint32_t b0 = __ldg(r0 + (c >> 5));
          const uint32_t b1 = __ldg(r1 + (c >> 5));
          fail = !((b0 & b1) >> (c & 31) & 1u);
        }
        const unsigned bal = __ballot_sync(FULL, fail);
        if (lane == 0) A.bitmap[w] = bal;
      }
      continue;
    }
    for (; w < we; ++w) {
      const uint32_t o = (uint32_t)(w - wbase) * 32 + lane;
      const bool valid = o < dsize;
      const uint32_t a = valid ? ldo(drv, o) : INF;
      uint32_t core = core0;
      if (core && !(core >> 31) && __shfl_sync(FULL, a, 0) < A.g.core_base) core = 0;  // word leaves the core
      bool fail = false;
#pragma unroll
      for (int q = 0; q < K - 1; ++q) {
        if (!((lists >> q) & 1u)) continue;
        bool found;
        if ((core >> q) & 1u) {
          // a is inside the step's [lo, hi): membership in the restricted list is edge existence
          found = valid && core_has_edge(A.g, d.owner[q], a);
        } else {
          const uint32_t* B = nbr + d.start[q];
          const uint32_t nb = d.len[q];
          if (nb <= 32) {
            found = warp_contains((uint32_t)lane < nb ? ldo(B, (uint32_t)lane) : INF, a);
          } else {
            // 32 splitters at (i+1)*step; lane's bucket by shuffle search, then a short per-lane search
            const uint32_t step = nb / 33u;
            const uint32_t sp = ldo(B, (uint32_t)(lane + 1) * step);
            int c = 0;
#pragma unroll
            for (int sh = 16; sh >= 1; sh >>= 1) {
              const uint32_t t = __shfl_sync(FULL, sp, c + sh - 1);
              if (t < a) c += sh;
            }
            c += __shfl_sync(FULL, sp, c) < a ? 1 : 0;  // c = #splitters < a, in [0, 32]
            const uint32_t lo = c ? (uint32_t)c * step + 1 : 0;
            const uint32_t hi = c < 32 ? (uint32_t)(c + 1) * step : nb;
            const uint32_t at = lb_thread(B, lo, hi, a);
            found = at < nb && ldo(B, at) == a;
          }
        }
        fail = fail || (found == (bool)((outs >> q) & 1u));
      }
      const unsigned bal = __ballot_sync(FULL, valid && fail);
      if (lane == 0) A.bitmap[w] = bal;
    }
  }
}

// Thread per sample, warp-uniform loop structure so survivor compaction can use
// one atomic per warp.
template <int K>
__global__ void __launch_bounds__(256) fr_pick_kernel(const FrontierArgs A, int s_step) {
  const uint32_t* __restrict__ nbr = A.g.nbr;
  const int lane = threadIdx.x & 31;
  const int j = s_step + 2;
  const bool reuse_next = s_step + 1 < K - 2 && A.step_reuse[s_step + 1];
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long base = (blockIdx.x * (unsigned long long)blockDim.x) + (threadIdx.x & ~31u);
       base < A.count; base += stride) {
    const unsigned long long i = base + lane;
    const bool act = i < A.count && A.work[i] != 0;
    Sample<K> S(A.seed, A.first_id + (act ? i : 0));
    bool alive = false;
    uint32_t o_pick = 0, nsurv = 0, lo2 = 0, hi2 = INF, pick = 0;
    const IsectDesc<K>* dp = reinterpret_cast<const IsectDesc<K>*>(A.desc) + (act ? i : 0);
    const uint32_t* words = A.bitmap + (act ? A.offsets[i] : 0);
    uint32_t ex[K];
    uint32_t dsize = 0;
    if (act) {
      load_state(A, i, S, j);
      dsize = dp->dsize;
      const uint32_t* D = dp->drv;
      uint32_t lo, hi;
      step_bounds(A.p, s_step, S, lo, hi);
      // bound vertices that survived the intersection are not candidates (walker.hpp:70-82)
#pragma unroll
      for (int q = 0; q < K; ++q) {
        ex[q] = INF;
        // the driver's own owner is never in it on a loop-free graph
        if (q < j && S.bnd[q] >= lo && S.bnd[q] < hi && !(A.g.loop_free && (uint32_t)q == dp->drv_pos)) {
          const uint32_t o = lb_thread(D, 0, dsize, S.bnd[q]);
          if (o < dsize && ldn(D, o) == S.bnd[q] && !((words[o >> 5] >> (o & 31)) & 1u)) ex[q] = o;
        }
      }
      const uint32_t nw = (dsize + 31) >> 5;
      auto live = [&](uint32_t w) -> unsigned {
        unsigned m = ~words[w];
        if (w == nw - 1 && (dsize & 31)) m &= (1u << (dsize & 31)) - 1u;
#pragma unroll
        for (int q = 0; q < K; ++q)
          if (ex[q] != INF && (ex[q] >> 5) == w) m &= ~(1u << (ex[q] & 31));
        return m;
      };
      unsigned long long cnt = 0;
      for (uint32_t w = 0; w < nw; ++w) cnt += __popc(live(w));
      if (cnt == 0) {
        finish(A, i, S, j, false);
      } else {
        unsigned long long r = S.rng.next_below(cnt);
        for (uint32_t w = 0; w < nw; ++w) {
          const unsigned m = live(w);
          const unsigned pc = __popc(m);
          if (r < pc) {
            o_pick = w * 32 + __fns(m, 0, (int)r + 1);
            break;
          }
          r -= pc;
        }
        S.alpha = __dmul_rn(S.alpha, (double)cnt);  // alpha *= |S_j| (ns_engine.cpp:39)
        pick = ldn(D, o_pick);
        if (dp->drv_pos != NO_DRV) {
#pragma unroll
          for (int q = 0; q < K; ++q)
            if ((uint32_t)q == dp->drv_pos) {  // lower_bound(pick + 1) = drv_rs + o + 1
              S.hbo[q] = dp->drv_rs + o_pick + 1;
              S.hbl[q] = pick + 1;
            }
        }
        bind(S, j, pick);
        if (AGPM_TWIN_HINT_MULTI && A.p.twin_hint[s_step] && A.g.twin && dp->drv_pos != NO_DRV) {  // position of v_drv in N(pick)
          uint32_t from = 0;
#pragma unroll
          for (int q = 0; q < K; ++q)
            if ((uint32_t)q == dp->drv_pos) from = S.bnd[q];
          S.hbo[j] = __ldg(A.g.twin + (unsigned long long)(D - nbr) + o_pick) + 1;
          S.hbl[j] = from + 1;
        }
        alive = true;
        if (reuse_next) {
          step_bounds(A.p, s_step + 1, S, lo2, hi2);
          for (uint32_t w = 0; w < nw; ++w) {
            unsigned m = live(w);
            while (m) {
              const uint32_t o = w * 32 + __ffs(m) - 1;
              m &= m - 1;
              const uint32_t x = ldn(D, o);
              nsurv += (o != o_pick && x >= lo2 && x < hi2) ? 1u : 0u;
            }
          }
        }
      }
    }
    // warp-aggregated allocation of the survivor lists
    uint32_t* surv = nullptr;
    if (reuse_next) {
      unsigned incl = nsurv;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const unsigned t = __shfl_up_sync(FULL, incl, d);
        if (lane >= d) incl += t;
      }
      unsigned long long wbase = 0;
      if (lane == 31 && incl) wbase = atomicAdd(A.surv_cursor + ((s_step + 1) & 1), (unsigned long long)incl);
      wbase = __shfl_sync(FULL, wbase, 31);
      const unsigned long long at = wbase + incl - nsurv;
      surv = A.survivors[(s_step + 1) & 1] + (at < A.surv_cap ? at : 0);
      if (alive && nsurv && at + nsurv <= A.surv_cap) {
        const uint32_t nw = (dsize + 31) >> 5;
        uint32_t k = 0;
        for (uint32_t w = 0; w < nw; ++w) {
          unsigned m = ~words[w];
          if (w == nw - 1 && (dsize & 31)) m &= (1u << (dsize & 31)) - 1u;
#pragma unroll
          for (int q = 0; q < K; ++q)
            if (ex[q] != INF && (ex[q] >> 5) == w) m &= ~(1u << (ex[q] & 31));
          while (m) {
            const uint32_t o = w * 32 + __ffs(m) - 1;
            m &= m - 1;
            const uint32_t x = ldn(dp->drv, o);
            if (o != o_pick && x >= lo2 && x < hi2) surv[k++] = x;
          }
        }
      }
    }
    if (alive) {
      if (reuse_next)
        advance<K>(A, i, S, s_step + 1, surv, nsurv);
      else
        advance<K>(A, i, S, s_step + 1, nullptr, 0);
    }
  }
}


// Nested survivor reuse is exact but, at word granularity, rarely cheaper than
// re-intersecting (a sample's step-j driver is ~1 bitmap word either way) while
// compaction makes the pick phase divergent; off unless enabled.
bool g_frontier_reuse = false;

// step s can reuse step s-1's survivors when its lists and bounds nest
bool nests(const DevPlan& p, int s) {
  if (s == 0) return false;
  const unsigned pin = p.in_mask[s - 1], pout = p.out_mask[s - 1], in = p.in_mask[s], out = p.out_mask[s];
  if ((pin & in) != pin || (pout & out) != pout) return false;
  if (__builtin_popcount(pin) == 1 && pout == 0) return false;  // previous step was single-list
  const unsigned prev_pos = 1u << (s + 1);                         // position bound by step s-1
  const bool lo_ok = p.gt_mask[s - 1] == 0 || (p.gt_mask[s] & prev_pos) ||
                     (p.gt_mask[s] & p.gt_mask[s - 1]) == p.gt_mask[s - 1];
  const bool hi_ok = p.lt_mask[s - 1] == 0 || (p.lt_mask[s] & prev_pos) ||
                     (p.lt_mask[s] & p.lt_mask[s - 1]) == p.lt_mask[s - 1];
  return lo_ok && hi_ok;
}

template <int K>
void run_frontier_k(const SampleLaunch& L, cudaStream_t s) {
  DeviceCtx& ctx = ctx_for_current_device();
  FrontierArgs A{};
  A.g = L.g;
  A.p = L.p;
  A.seed = L.seed;
  for (int st = 0; st < K - 2; ++st) {
    const unsigned in_m = L.p.in_mask[st], out_m = L.p.out_mask[st];
    A.step_multi[st] = !(__builtin_popcount(in_m) == 1 && out_m == 0);
    A.step_reuse[st] = g_frontier_reuse && A.step_multi[st] && nests(L.p, st);
  }
  const unsigned long long cap = std::min<unsigned long long>(L.count, kFrontierCap);
  A.cap = cap;
  size_t bytes = 0;
  auto carve = [&](size_t n) {
    size_t at = (bytes + 255) & ~size_t(255);
    bytes = at + n;
    return at;
  };
  const size_t o_ctr = carve(8 * cap), o_alpha = carve(8 * cap), o_bnd = carve(4ull * K * cap),
               o_hbo = carve(4ull * K * cap), o_hbl = carve(4ull * K * cap), o_work = carve(8 * (cap + 1)),
               o_off = carve(8 * (cap + 1)), o_desc = carve(sizeof(IsectDesc<K>) * cap), o_cur = carve(64);
  size_t scan_tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_tmp, (const unsigned long long*)nullptr,
                                (unsigned long long*)nullptr, (int64_t)cap + 1, s);
  const size_t o_tmp = carve(scan_tmp + 256);
  char* slab = static_cast<char*>(ctx.get(9, bytes));
  A.ctr = reinterpret_cast<unsigned long long*>(slab + o_ctr);
  A.alpha = reinterpret_cast<double*>(slab + o_alpha);
  A.bnd = reinterpret_cast<uint32_t*>(slab + o_bnd);
  A.hbo = reinterpret_cast<uint32_t*>(slab + o_hbo);
  A.hbl = reinterpret_cast<uint32_t*>(slab + o_hbl);
  A.work = reinterpret_cast<unsigned long long*>(slab + o_work);
  A.offsets = reinterpret_cast<unsigned long long*>(slab + o_off);
  A.desc = slab + o_desc;
  A.surv_cursor = reinterpret_cast<unsigned long long*>(slab + o_cur);
  void* tmp = slab + o_tmp;
  auto* h_total = static_cast<unsigned long long*>(ctx.get_pinned(2, 64));
  bool any_reuse = false;
  for (int st = 0; st < K - 2; ++st) any_reuse = any_reuse || A.step_reuse[st];

  const int sms = ctx.sm_count;
  for (unsigned long long done = 0; done < L.count; done += cap) {
    const unsigned long long c = std::min(cap, L.count - done);
    A.count = c;
    A.first_id = L.first_id + done;
    A.values = L.values + done;
    A.bindings = L.bindings ? L.bindings + done * K : nullptr;
    const unsigned blocks = (unsigned)std::min<unsigned long long>((c + 255) / 256, (unsigned long long)sms * 16);
    fr_seed_kernel<K><<<blocks, 256, 0, s>>>(A);
    count_launch();
    AGPM_CUDA(cudaGetLastError());
    for (int st = 0; st < K - 2; ++st) {
      if (!A.step_multi[st]) continue;
      AGPM_CUDA(cudaMemsetAsync(A.work + c, 0, 8, s));
      size_t tb = scan_tmp;
      AGPM_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, A.work, A.offsets, (int64_t)c + 1, s));
      AGPM_CUDA(cudaMemcpyAsync(h_total, A.offsets + c, 8, cudaMemcpyDeviceToHost, s));
      AGPM_CUDA(cudaStreamSynchronize(s));
      const unsigned long long words = *h_total;
      if (words) {
        A.bitmap = static_cast<uint32_t*>(ctx.get(8, 4 * words + 64));
        if (any_reuse) {  // survivors <= driver elements <= 32 * words
          A.surv_cap = 32 * words;
          const int slot = (st + 1) & 1;
          A.survivors[slot] = static_cast<uint32_t*>(ctx.get(10 + slot, 4 * A.surv_cap + 64));
          AGPM_CUDA(cudaMemsetAsync(A.surv_cursor + slot, 0, 8, s));
        }
        const unsigned long long warps = std::min<unsigned long long>(words, (unsigned long long)sms * 64);
        fr_isect_kernel<K><<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(A, words);
        count_launch();
        AGPM_CUDA(cudaGetLastError());
      }
      fr_pick_kernel<K><<<blocks, 256, 0, s>>>(A, st);
      count_launch();
      AGPM_CUDA(cudaGetLastError());
    }
  }
}



}  // namespace

void set_frontier_reuse(bool on) { g_frontier_reuse = on; }


void launch_ns_frontier(const SampleLaunch& L, cudaStream_t s) {
  if (L.bytes_out) throw std::invalid_argument("B_min accounting runs on the warp sampler");
#define AGPM_K(KK)            \
  case KK:                    \
    run_frontier_k<KK>(L, s); \
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
