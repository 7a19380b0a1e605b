// 4-cycles touching the sparse region of a degree-relabelled graph — the exact
// C_sparse of the region split for the "4cycle" plan (config 3), without
// enumerating wedges through hubs one by one.
//
// C_sparse counts every 4-cycle whose minimum vertex m lies in V_s = [0, tau_id)
// once (the rooted exact count, exact_engine.cpp:19-62 with roots < tau_id).
// With m's two cycle neighbours b < d (both > m, both in N+(m)) and the
// opposite vertex c in N(b) ∩ N(d), c > m:
//
//   C_sparse = sum_{m < tau_id} sum_{b<d in N+(m)} |N(b) ∩ N(d) ∩ (m, inf)|.
//
// Group the terms by the pair (b, d). Its sparse middles K = {m in N(b)∩N(d) :
// m < min(b, tau_id)} are exactly the common neighbours below min(b, tau_id),
// so the i-th smallest one sees s - i common neighbours above it (s = |N(b) ∩
// N(d)|) and the pair contributes  k*s - k(k+1)/2,  k = |K|. The work splits by
// where b falls relative to the pair core [cb, n) (the top P <= 65 536 ids, all
// dense: cb >= tau_id):
//
//  * b, d both in the pair core (the hub pairs that make the wedge DFS slow):
//    one pass over the NON-core middles m < cb adds, for every pair of m's
//    pair-core neighbours, 1 to s_low(b, d) and (m < tau_id) to k(b, d) — a
//    packed u64 atomic into a triangular P x P table; the pair-core middles'
//    share of s is the popcount of the AND of b's and d's dense-core bit rows
//    (core_bits.cu) over the pair-core columns.
//    Then k*s - k(k+1)/2 per table entry with k > 0.
//  * b below the pair core: per sparse wedge (m; b, d) directly, the count of
//    c in N(b) ∩ (m, inf) adjacent to d (one core bit, or a search of the
//    shorter list) — N(b) is a short list here.
//
// Exact integer arithmetic throughout; tests/test_gpu_region.py pins it to the
// wedge-DFS rooted count and to exact(G) - exact(G[V_d]).
#include <cub/cub.cuh>

#include <algorithm>
#include <stdexcept>

#include "device.cuh"
#include "ns_common.cuh"

namespace agpm_b200 {

namespace {

constexpr int kC4Threads = 256;

struct C4Args {
  const VtxInfo* __restrict__ vtx;
  const uint32_t* __restrict__ nbr;
  const uint32_t* __restrict__ core;  // dense-core bit matrix, rows of wpr words, ids >= core_base
  uint32_t core_base, wpr;
  uint32_t n, tau_id, cb, P;
  unsigned long long* __restrict__ table;  // P(P-1)/2 packed (k << 32 | s_low), column d' holds b' < d'
  unsigned long long* __restrict__ total;
  unsigned long long* __restrict__ cursor;
};

__device__ __forceinline__ unsigned long long tri(uint32_t b, uint32_t d) {  // b < d, both pair-core local
  return (unsigned long long)d * (d - 1) / 2 + b;
}

__device__ __forceinline__ bool has_edge_dev(const C4Args& A, uint32_t x, uint32_t y) {
  if (A.core && x >= A.core_base && y >= A.core_base) {
    const uint32_t c = y - A.core_base;
    return (__ldg(A.core + (unsigned long long)(x - A.core_base) * A.wpr + (c >> 5)) >> (c & 31)) & 1u;
  }
  const VtxInfo vx = load_vtx(A.vtx, x), vy = load_vtx(A.vtx, y);
  const bool sx = vx.deg <= vy.deg;  // search the shorter list
  const unsigned long long b = sx ? vx.begin : vy.begin, e = b + (sx ? vx.deg : vy.deg);
  const uint32_t t = sx ? y : x;
  const unsigned long long at = lower_bound_dev(A.nbr, b, e, t);
  return at < e && ldn(A.nbr, at) == t;
}

// pass 1: warp per non-core middle m; every pair of its pair-core neighbours
__global__ void __launch_bounds__(kC4Threads) c4_pairs_kernel(C4Args A) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned long long m = 0;
    if (lane == 0) m = atomicAdd(A.cursor, 1ull);
    m = __shfl_sync(FULL, m, 0);
    if (m >= A.cb) return;
    const VtxInfo vi = load_vtx(A.vtx, (uint32_t)m);
    // core neighbours: the suffix of N(m) from lower_bound(cb)
    const unsigned long long b0 = lower_bound_dev(A.nbr, vi.begin, vi.begin + vi.deg, A.cb);
    const uint32_t len = (uint32_t)(vi.begin + vi.deg - b0);
    if (len < 2) continue;
    const unsigned long long add = m < A.tau_id ? (1ull << 32) | 1ull : 1ull;
    for (uint32_t i = 0; i + 1 < len; ++i) {
      const uint32_t bl = ldn(A.nbr, b0 + i) - A.cb;
      for (uint32_t j = i + 1 + lane; j < len; j += 32) {
        const uint32_t dl = ldn(A.nbr, b0 + j) - A.cb;
        atomicAdd(A.table + tri(bl, dl), add);
      }
    }
  }
}

// pass 2: block per pair-core column d'; entries b' < d' with k > 0 contribute
// k*s - k(k+1)/2, s = s_low + popcount(row_b & row_d) over the dense core
__global__ void __launch_bounds__(kC4Threads) c4_table_kernel(C4Args A) {
  extern __shared__ uint32_t srow[];  // row of d, A.wpr words
  __shared__ uint32_t q_b[kC4Threads];
  __shared__ unsigned long long q_v[kC4Threads];
  __shared__ int q_n;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned long long acc = 0;
  for (uint32_t dl = blockIdx.x + 1; dl < A.P; dl += gridDim.x) {
    const uint32_t d = A.cb + dl;
    const uint32_t* rd = A.core + (unsigned long long)(d - A.core_base) * A.wpr;
    for (uint32_t w = threadIdx.x; w < A.wpr; w += blockDim.x) srow[w] = __ldg(rd + w);
    const unsigned long long col = tri(0, dl);
    for (uint32_t c0 = 0; c0 < dl; c0 += blockDim.x) {
      if (threadIdx.x == 0) q_n = 0;
      __syncthreads();
      const uint32_t bl = c0 + threadIdx.x;
      if (bl < dl) {
        const unsigned long long v = A.table[col + bl];
        if (v >> 32) {
          const int at = atomicAdd(&q_n, 1);
          q_b[at] = bl;
          q_v[at] = v;
        }
      }
      __syncthreads();
      for (int it = wid; it < q_n; it += kC4Threads / 32) {
        const uint32_t b = A.cb + q_b[it];
        const uint32_t* rb = A.core + (unsigned long long)(b - A.core_base) * A.wpr;
        // common neighbours inside the pair core only (columns >= cb): those below
        // cb are the non-core middles pass 1 already counted
        const uint32_t o = A.cb - A.core_base, w0 = o >> 5;
        unsigned long long pc = 0;
        for (uint32_t w = w0 + lane; w < A.wpr; w += 32) {
          uint32_t x = __ldg(rb + w) & srow[w];
          if (w == w0) x &= ~0u << (o & 31);
          pc += __popc(x);
        }
#pragma unroll
        for (int sh = 16; sh > 0; sh >>= 1) pc += __shfl_xor_sync(FULL, pc, sh);
        if (lane == 0) {
          const unsigned long long k = q_v[it] >> 32, s = (q_v[it] & 0xffffffffull) + pc;
          acc += k * s - k * (k + 1) / 2;
        }
      }
      __syncthreads();
    }
  }
  if (acc) atomicAdd(A.total, acc);
}

// pass 3: warp per sparse m; wedges (m; b, d), b < d in N+(m), b below the pair
// core: lanes take c in N(b) ∩ (m, inf) and test c ~ d for every such d
__global__ void __launch_bounds__(kC4Threads) c4_direct_kernel(C4Args A) {
  const int lane = threadIdx.x & 31;
  unsigned long long acc = 0;
  for (;;) {
    unsigned long long m = 0;
    if (lane == 0) m = atomicAdd(A.cursor, 1ull);
    m = __shfl_sync(FULL, m, 0);
    if (m >= A.tau_id) break;
    const VtxInfo vm = load_vtx(A.vtx, (uint32_t)m);
    const unsigned long long u0 = vm.begin + vm.up, u1 = vm.begin + vm.deg;  // N+(m) = ids > m
    for (unsigned long long ib = u0; ib + 1 < u1; ++ib) {
      const uint32_t b = ldn(A.nbr, ib);
      if (b >= A.cb) break;  // the rest pair inside the pair core (pass 1/2)
      const VtxInfo vb = load_vtx(A.vtx, b);
      const unsigned long long c0 = lower_bound_dev(A.nbr, vb.begin, vb.begin + vb.deg, (uint32_t)m + 1);
      const unsigned long long c1 = vb.begin + vb.deg;
      for (unsigned long long cc = c0; cc < c1; cc += 32) {
        const bool valid = cc + lane < c1;
        const uint32_t c = valid ? ldn(A.nbr, cc + lane) : 0u;
        for (unsigned long long id = ib + 1; id < u1; ++id) {
          const uint32_t d = ldn(A.nbr, id);
          if (valid && c != d && has_edge_dev(A, c, d)) ++acc;
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
  if (lane == 0 && acc) atomicAdd(A.total, acc);
}

}  // namespace

bool plan_is_plain_4cycle(const agpm_plan* p) {
  if (p->k != 4 || p->n_edges != 4 || p->induced || p->verify_mode != 0 || !p->symmetry_enabled) return false;
  for (int v = 0; v < 4; ++v)
    if (__builtin_popcount(p->adjacency[v]) != 2) return false;
  return true;
}

// C_sparse of the 4-cycle region split; g: plain symmetric degree-relabelled view
unsigned long long cycle4_sparse_count(agpm_graph* g, uint32_t tau_id, cudaStream_t s) {
  if (!g->plain || g->oriented) throw std::invalid_argument("4-cycle sparse count needs a plain symmetric view");
  DeviceCtx& ctx = ctx_for_current_device();
  ensure_core_bits(g, s);
  C4Args A{};
  A.vtx = g->vtx;
  A.nbr = g->nbr;
  A.core = g->core;
  A.core_base = g->core_base;
  A.wpr = g->core_wpr;
  A.n = g->n;
  A.tau_id = std::min(tau_id, g->n);
  // pair core: the top P ids, inside the dense-core matrix and above V_s;
  // the triangular table costs 4 P^2 bytes, so P shrinks if HBM is short
  uint32_t P = g->core ? std::min({65536u, g->core_dim, g->n - A.tau_id}) : 0u;
  size_t free_b = 0, total_b = 0;
  AGPM_CUDA(cudaMemGetInfo(&free_b, &total_b));
  while (P > 1 && 4ull * P * P > free_b / 2) P /= 2;
  if (P < 2) P = 0;
  A.P = P;
  A.cb = g->n - P;
  auto* scratch = static_cast<unsigned long long*>(ctx.get(3, 64));
  A.total = scratch;
  A.cursor = scratch + 1;
  AGPM_CUDA(cudaMemsetAsync(scratch, 0, 16, s));
  const unsigned blocks = (unsigned)ctx.sm_count * (2048 / kC4Threads);
  if (P) {
    const unsigned long long entries = (unsigned long long)P * (P - 1) / 2;
    unsigned long long* table = nullptr;
    AGPM_CUDA(dev_malloc(&table, 8ull * entries));
    A.table = table;
    AGPM_CUDA(cudaMemsetAsync(A.table, 0, 8ull * entries, s));
    c4_pairs_kernel<<<blocks, kC4Threads, 0, s>>>(A);
    count_launch();
    AGPM_CUDA(cudaGetLastError());
    const size_t shmem = 4ull * A.wpr;
    if (shmem > 48 * 1024)
      AGPM_CUDA(cudaFuncSetAttribute(c4_table_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shmem));
    c4_table_kernel<<<std::min<unsigned>(blocks, P), kC4Threads, shmem, s>>>(A);
    count_launch();
    AGPM_CUDA(cudaGetLastError());
  }
  AGPM_CUDA(cudaMemsetAsync(A.cursor, 0, 8, s));
  c4_direct_kernel<<<blocks, kC4Threads, 0, s>>>(A);
  count_launch();
  AGPM_CUDA(cudaGetLastError());
  unsigned long long h = 0;
  AGPM_CUDA(cudaMemcpyAsync(&h, A.total, 8, cudaMemcpyDeviceToHost, s));
  AGPM_CUDA(cudaStreamSynchronize(s));
  if (A.table) AGPM_CUDA(dev_free(A.table));
  return h;
}

}  // namespace agpm_b200
