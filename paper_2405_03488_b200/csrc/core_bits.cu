// Dense-core adjacency bit matrix for the frontier intersections.
//
// On a degree-relabelled graph the highest ids are the highest-degree
// vertices, and eager-verify candidates always sit above the bound vertices'
// ids for clique-like steps — so most membership tests "a in N(w)" of the
// intersection phase have both a and w among the top ids. For the top C ids
// (the "core", default C = 65536 -> a 512 MB matrix; its hot rows stay in the 126 MB L2)
// the adjacency is kept as a C x C bit matrix: a core test is ONE L2 word load
// per lane instead of a splitter load, a shuffle search and a dependent
// per-lane search. On config 2, 92 % / 97.7 % of the isect membership tests
// fall inside a 16 K / 32 K core, and one 2^24-sample 4-clique launch drops
// from 27.2 ms to 15.9 ms (profiles/r1/README.md). With the flat sampler a
// 64 K core beats 32 K on every RMAT scale measured (20: 8.8 vs 9.4 ms, 22:
// 15.1 vs 17.0, 24: 26.4 vs 36.2, 27: 79.5 vs 91.8 ms per 2^24 4-clique samples).
//
// Exact by construction (it is the adjacency restricted to [base, n)), so it
// changes no result; it only replaces how membership is answered.
#include <algorithm>

#include <atomic>

#include "device.cuh"
#include "ns_common.cuh"

namespace agpm_b200 {
namespace {

constexpr uint32_t kCoreAuto = 0xffffffffu;
std::atomic<uint32_t> g_core_dim{kCoreAuto};

// one block per core row: the row is built in shared memory (zeroed, one
// shared atomic per core neighbour) and written out with 16-B stores
__global__ void __launch_bounds__(256) core_rows_kernel(const VtxInfo* __restrict__ vtx,
                                                        const uint32_t* __restrict__ nbr, uint32_t base,
                                                        uint32_t rows, uint32_t wpr, uint32_t* __restrict__ bits) {
  extern __shared__ uint32_t row[];
  __shared__ uint32_t s_start;
  const int lane = threadIdx.x & 31;
  for (uint32_t r = blockIdx.x; r < rows; r += gridDim.x) {
    for (uint32_t i = threadIdx.x; i < wpr; i += blockDim.x) row[i] = 0;
    const VtxInfo vi = load_vtx(vtx, base + r);
    const uint32_t* list = nbr + vi.begin;
    if (threadIdx.x < 32) {
      const uint32_t start = kary_lb(list, 0, vi.deg, base, lane, nullptr);
      if (lane == 0) s_start = start;
    }
    __syncthreads();
    for (uint32_t i = s_start + threadIdx.x; i < vi.deg; i += blockDim.x) {
      const uint32_t c = __ldg(list + i) - base;
      atomicOr(row + (c >> 5), 1u << (c & 31));
    }
    __syncthreads();
    uint32_t* out = bits + (unsigned long long)r * wpr;
    if ((wpr & 3) == 0) {
      const uint4* src = reinterpret_cast<const uint4*>(row);
      uint4* dst = reinterpret_cast<uint4*>(out);
      for (uint32_t i = threadIdx.x; i < wpr / 4; i += blockDim.x) dst[i] = src[i];
    } else {
      for (uint32_t i = threadIdx.x; i < wpr; i += blockDim.x) out[i] = row[i];
    }
    __syncthreads();
  }
}

// one thread per arc (u -> v): lower_bound of u in N(v) (u is there: symmetric view)
__global__ void twin_kernel(const VtxInfo* __restrict__ vtx, const uint32_t* __restrict__ nbr,
                            const unsigned long long* __restrict__ seed_arcs, unsigned long long arcs,
                            uint32_t* __restrict__ twin) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < arcs;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long a = __ldg(seed_arcs + i);
    const uint32_t u = (uint32_t)(a >> 32), v = (uint32_t)a;
    const VtxInfo vv = load_vtx(vtx, v);
    unsigned long long lo = vv.begin, hi = vv.begin + vv.deg;
    while (lo < hi) {
      const unsigned long long mid = (lo + hi) >> 1;
      if (__ldg(nbr + mid) < u)
        lo = mid + 1;
      else
        hi = mid;
    }
    twin[i] = (uint32_t)(lo - vv.begin);
  }
}

}  // namespace

// The twin index is a speed hint (identical samples without it): it is built
// best-effort — skipped when HBM is short (4 B per arc, 16.9 GB on RMAT-27) —
// and published only once its build kernel has finished, under the view's
// index lock, so no launch on any stream or host thread can see a pointer to
// an index still being written.
void ensure_twin_arcs(agpm_graph* g, cudaStream_t s) {
  if (g->twin || !g->plain || g->oriented || g->arcs == 0) return;
  std::lock_guard<std::mutex> lk(g->index_mu);
  if (g->twin) return;
  const size_t need = 4ull * g->arcs;
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess || free_b < need + (2ull << 30)) {
    cudaGetLastError();
    return;
  }
  uint32_t* tw = nullptr;
  if (dev_malloc(&tw, need) != cudaSuccess) {
    cudaGetLastError();  // out of memory: sample without the hint
    return;
  }
  DeviceCtx& ctx = ctx_for_current_device();
  const unsigned blocks = (unsigned)std::min<unsigned long long>((g->arcs + 255) / 256, (unsigned long long)ctx.sm_count * 16);
  twin_kernel<<<blocks, 256, 0, s>>>(g->vtx, g->nbr, g->seed_arcs, g->arcs, tw);
  count_launch();
  AGPM_CUDA(cudaGetLastError());
  AGPM_CUDA(cudaStreamSynchronize(s));
  g->bytes += need;
  g->twin = tw;
}

void set_core_dim(uint32_t dim) { g_core_dim = dim; }
uint32_t core_dim_setting() { return g_core_dim; }

// Core dimension for a view. Auto: 65 536 up to 2^21 vertices; 262 144 up to 2^25
// and 524 288 above, where hub rows outside a smaller core are common — measured per
// 2^24 samples, 64 K -> 256 K core: RMAT-27 4-clique 41.8 -> 29.8 ms, 4-cycle 39.2 ->
// 29.1, RMAT-22 4-clique (flat) 13.2 -> 12.0, 4-cycle 11.2 -> 10.3, while RMAT-20 gains
// < 1 % for a matrix 16x larger (rebuilt with every fresh view); 256 K -> 512 K core:
// RMAT-27 4-clique frontier 29.7 -> 28.0 ms, flat 39.8 -> 31.6; RMAT-26 flat 25.4 -> 22.3
// (frontier 24.0 -> 24.3). The larger matrices (8 GB / 32 GB) are only taken when
// they leave most of the device free.
uint32_t core_dim_for(const agpm_graph* g) {
  const uint32_t set = g_core_dim.load();
  if (set != kCoreAuto) return std::min(set, g->n);
  uint32_t dim = g->n > (1u << 25) ? 524288u : g->n > (1u << 21) ? 262144u : 65536u;
  if (dim > 65536u) {
    // blocks the stream-ordered pool still caches (ingest temporaries) count as free
    size_t free_b = 0, total_b = 0;
    cudaMemPool_t pool;
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      size_t reserved = 0, used = 0;
      if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved) == cudaSuccess &&
          cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess && reserved > used)
        free_b = reserved - used;
    }
    size_t dev_free_b = 0;
    if (cudaMemGetInfo(&dev_free_b, &total_b) == cudaSuccess) {
      free_b += dev_free_b;
    } else {
      cudaGetLastError();
      free_b = 0;
    }
    while (dim > 65536u && (size_t)dim * dim / 8 > free_b / 3) dim /= 2;
    if (dim < 262144u) dim = 65536u;
  }
  return std::min(dim, g->n);
}

// Published after its build finished, under the view's index lock (see ensure_twin_arcs).
void ensure_core_bits(agpm_graph* g, cudaStream_t s) {
  const bool autodim = g_core_dim.load() == kCoreAuto;
  if (g->core && autodim && g->core_auto) return;  // the auto choice is made once per view
  const uint32_t want = g->oriented || !g->plain ? 0u : core_dim_for(g);
  if (g->core && g->core_dim == want) return;
  std::lock_guard<std::mutex> lk(g->index_mu);
  if (g->core && g->core_dim == want) return;
  if (g->core) {
    AGPM_CUDA(cudaStreamSynchronize(s));
    AGPM_CUDA(dev_free(g->core));
    g->bytes -= 4ull * g->core_wpr * g->core_dim;
    g->core = nullptr;
    g->core_dim = g->core_wpr = g->core_base = 0;
  }
  if (want == 0) return;
  DeviceCtx& ctx = ctx_for_current_device();
  const uint32_t base = g->n - want;
  const uint32_t wpr = (want + 31) / 32;
  uint32_t* bits = nullptr;
  AGPM_CUDA(dev_malloc(&bits, 4ull * wpr * want));
  const size_t shmem = 4ull * wpr;
  if (shmem > 48 * 1024)
    AGPM_CUDA(cudaFuncSetAttribute(core_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shmem));
  const unsigned blocks = std::max(1u, std::min(want, (unsigned)ctx.sm_count * 8));
  core_rows_kernel<<<blocks, 256, shmem, s>>>(g->vtx, g->nbr, base, want, wpr, bits);
  count_launch();
  AGPM_CUDA(cudaGetLastError());
  AGPM_CUDA(cudaStreamSynchronize(s));
  g->core = bits;
  g->core_base = base;
  g->core_wpr = wpr;
  g->core_dim = want;
  g->core_auto = autodim;
  g->bytes += 4ull * wpr * want;
}

}  // namespace agpm_b200

using namespace agpm_b200;

extern "C" int agpm_graph_prepare(agpm_graph* g, void* stream) {
  // build a view's sampling indexes now (dense-core bit matrix at the configured
  // dimension, twin arcs) instead of lazily (first launch / after `arcs` sampled ids) — e.g.
  // on an upload thread, overlapped with sampling of another view
  return guarded([&] {
    if (!g) throw std::invalid_argument("null argument");
    DeviceGuard guard(g->device);
    cudaStream_t s = pick_stream(stream);
    ensure_core_bits(g, s);
    ensure_twin_arcs(g, s);
  });
}

extern "C" int agpm_ns_set_core_dim(uint32_t dim) {
  return guarded([&] {
    // 0xffffffff = auto, see core_dim_for; the build kernel keeps one row (dim / 8 bytes)
    // in shared memory
    if (dim > 1048576 && dim != kCoreAuto) throw std::invalid_argument("core dimension must be <= 1048576");
    set_core_dim(dim);
  });
}
