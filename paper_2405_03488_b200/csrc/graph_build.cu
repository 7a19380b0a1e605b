// GPU graph ingest: edge generation, symmetrise / dedup, degree relabel, CSR
// build and orientation entirely in HBM (SURVEY §8(f) "next": the data format
// on the input side of the sampling path).
//
// The reference builds its CSR on the host (csr_graph.cpp:46-72
// build_from_edges: normalise u<v, drop loops, sort + unique, emit both arcs,
// ascending lists; test_graphs.hpp RMAT generator; relabel / orientation in
// csr_graph.cpp). Here every stage is a device pass over u64 keys:
//
//   edges   key = min<<32 | max   (self-loops -> ~0, sorted to the end)
//   sort    cub::DeviceRadixSort (64-bit num_items; RMAT-27 = 2.1e9 keys)
//   unique  cub::DeviceSelect::Unique, sentinel dropped
//   relabel degree histogram (atomics), stable radix sort of (degree, id) =
//           rank of (degree, id) — the same order as host relabel_by_degree
//   arcs    two arc keys u<<32|v per edge in the new ids, radix-sorted: the
//           sorted arc keys ARE seed_arcs[] (arc-index order), nbr[] is their
//           low word, and the vertex boundaries give begin[] — no second pass
//           over the lists.
//
// Output graphs are bit-identical to the host builders (graph_from_edges,
// gen_rmat, gen_er_fast, relabel_by_degree, orient_by_degree); the GPU suite
// checks that by downloading both.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "device.cuh"
#include "rng.cuh"

namespace agpm_b200 {
namespace {

constexpr unsigned long long kLoop = ~0ull;

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  void alloc(size_t count) {
    release();
    n = count;
    AGPM_CUDA(dev_malloc(&p, sizeof(T) * (count ? count : 1)));
  }
  void release() {
    if (p) dev_free(p);
    p = nullptr;
    n = 0;
  }
  T* take() {
    T* q = p;
    p = nullptr;
    n = 0;
    return q;
  }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

int grid_for(uint64_t items, int sm_count, int block = 256) {
  uint64_t want = (items + block - 1) / block;
  uint64_t cap = (uint64_t)sm_count * 16;
  return (int)std::max<uint64_t>(1, std::min(want, cap));
}

// ------------------------------------------------------------------ generators
// test_graphs.hpp RMAT recursion, one CounterRng(seed, "rmat", i) per edge
// (host twin: host_graph.cpp gen_rmat).
__global__ void rmat_kernel(uint32_t scale, double a, double ab, double abc, uint64_t seed, uint64_t m,
                            unsigned long long* __restrict__ keys) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    CounterRng rng(seed, 0x726d6174ull, i);
    uint32_t u = 0, v = 0;
    for (uint32_t l = 0; l < scale; ++l) {
      double r = rng.next_double();
      uint32_t bu = 0, bv = 0;
      if (r < a) {
      } else if (r < ab) {
        bv = 1;
      } else if (r < abc) {
        bu = 1;
      } else {
        bu = 1;
        bv = 1;
      }
      u = (u << 1) | bu;
      v = (v << 1) | bv;
    }
    keys[i] = u == v ? kLoop : ((unsigned long long)min(u, v) << 32) | max(u, v);
  }
}

// host_graph.cpp gen_er_fast: endpoints uniform by CounterRng(seed, "er", i)
__global__ void er_kernel(uint32_t n, uint64_t seed, uint64_t m, unsigned long long* __restrict__ keys) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    CounterRng rng(seed, 0x6572ull, i);
    uint32_t u = (uint32_t)rng.next_below(n);
    uint32_t v = (uint32_t)rng.next_below(n);
    keys[i] = u == v ? kLoop : ((unsigned long long)min(u, v) << 32) | max(u, v);
  }
}

// host edge pairs (u0, v0, u1, v1, ...) already copied to the device
__global__ void pairs_kernel(const uint32_t* __restrict__ pairs, uint64_t m, unsigned long long* __restrict__ keys,
                             unsigned int* __restrict__ max_id) {
  unsigned int local = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t u = pairs[2 * i], v = pairs[2 * i + 1];
    local = max(local, max(u, v));
    keys[i] = u == v ? kLoop : ((unsigned long long)min(u, v) << 32) | max(u, v);
  }
  for (int o = 16; o; o >>= 1) local = max(local, __shfl_xor_sync(0xffffffffu, local, o));
  if ((threadIdx.x & 31) == 0 && local) atomicMax(max_id, local);
}

// ------------------------------------------------------------------ CSR stages
__global__ void degree_kernel(const unsigned long long* __restrict__ edges, uint64_t m,
                              unsigned int* __restrict__ deg) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    unsigned long long k = edges[i];
    atomicAdd(&deg[(uint32_t)(k >> 32)], 1u);
    atomicAdd(&deg[(uint32_t)k], 1u);
  }
}

__global__ void iota_kernel(uint32_t n, uint32_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (uint32_t)i;
}

__global__ void invert_kernel(const uint32_t* __restrict__ order, uint32_t n, uint32_t* __restrict__ new_id) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    new_id[order[i]] = (uint32_t)i;
}

// both arcs of every undirected edge, endpoints mapped through new_id (or not)
__global__ void expand_kernel(const unsigned long long* __restrict__ edges, uint64_t m,
                              const uint32_t* __restrict__ new_id, unsigned long long* __restrict__ arcs) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    unsigned long long k = edges[i];
    uint32_t u = (uint32_t)(k >> 32), v = (uint32_t)k;
    if (new_id) {
      u = new_id[u];
      v = new_id[v];
    }
    arcs[2 * i] = ((unsigned long long)u << 32) | v;
    arcs[2 * i + 1] = ((unsigned long long)v << 32) | u;
  }
}

// arcs of an existing view, relabelled (both directions are already present)
__global__ void remap_arcs_kernel(const unsigned long long* __restrict__ in, uint64_t count,
                                  const uint32_t* __restrict__ new_id, unsigned long long* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x) {
    unsigned long long k = in[i];
    out[i] = ((unsigned long long)new_id[(uint32_t)(k >> 32)] << 32) | new_id[(uint32_t)k];
  }
}

__global__ void view_degree_kernel(const VtxInfo* __restrict__ vtx, uint32_t n, unsigned int* __restrict__ deg) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    deg[i] = vtx[i].deg;
}

// orientation flag: keep arc (u, v) iff (deg u, u) < (deg v, v)  (csr_graph.cpp orient)
struct OrientKeep {
  const VtxInfo* vtx;
  __device__ bool operator()(unsigned long long k) const {
    uint32_t u = (uint32_t)(k >> 32), v = (uint32_t)k;
    unsigned int du = vtx[u].deg, dv = vtx[v].deg;
    return du < dv || (du == dv && u < v);
  }
};

// Vertex boundaries of sorted arc keys: first[u] = index of u's first arc,
// last[u] = one past its last; untouched (zero-degree) vertices keep 0/0.
__global__ void bounds_kernel(const unsigned long long* __restrict__ arcs, uint64_t count,
                              unsigned long long* __restrict__ first, unsigned long long* __restrict__ last,
                              uint32_t* __restrict__ nbr) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x) {
    unsigned long long k = arcs[i];
    uint32_t u = (uint32_t)(k >> 32);
    nbr[i] = (uint32_t)k;
    if (i == 0 || (uint32_t)(arcs[i - 1] >> 32) != u) first[u] = i;
    if (i + 1 == count || (uint32_t)(arcs[i + 1] >> 32) != u) last[u] = i + 1;
  }
}

__global__ void deg_from_bounds_kernel(const unsigned long long* __restrict__ first,
                                       const unsigned long long* __restrict__ last, uint32_t n,
                                       unsigned long long* __restrict__ deg) {
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < n;
       u += (uint64_t)gridDim.x * blockDim.x)
    deg[u] = last[u] - first[u];
}

__global__ void vtx_from_bounds_kernel(const unsigned long long* __restrict__ begin, const uint32_t* __restrict__ nbr,
                                       uint32_t n, VtxInfo* __restrict__ vtx) {
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < n;
       u += (uint64_t)gridDim.x * blockDim.x) {
    unsigned long long b = begin[u], e = begin[u + 1];
    unsigned long long lo = b, hi = e;
    while (lo < hi) {  // up = #neighbours <= u
      unsigned long long mid = (lo + hi) >> 1;
      if (nbr[mid] <= (uint32_t)u)
        lo = mid + 1;
      else
        hi = mid;
    }
    VtxInfo v;
    v.begin = b;
    v.deg = (unsigned int)(e - b);
    v.up = (unsigned int)(lo - b);
    vtx[u] = v;
  }
}

int bits_for(uint64_t x) {
  int b = 0;
  while (b < 64 && (x >> b)) ++b;
  return std::max(b, 1);
}

void sort_keys(DevBuf<unsigned long long>& keys, DevBuf<unsigned long long>& alt, uint64_t count, int end_bit,
               cudaStream_t s) {
  if (count < 2) {
    return;
  }
  if (alt.n < count) alt.alloc(count);
  cub::DoubleBuffer<unsigned long long> db(keys.p, alt.p);
  size_t tmp = 0;
  AGPM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, db, (int64_t)count, 0, end_bit, s));
  DevBuf<unsigned char> t(tmp + 16);
  AGPM_CUDA(cub::DeviceRadixSort::SortKeys(t.p, tmp, db, (int64_t)count, 0, end_bit, s));
  if (db.Current() != keys.p) std::swap(keys.p, alt.p), std::swap(keys.n, alt.n);
  AGPM_CUDA(cudaStreamSynchronize(s));
}

// sorted keys -> unique keys (in `out`), sentinel loops dropped; returns count
uint64_t unique_edges(DevBuf<unsigned long long>& keys, uint64_t count, DevBuf<unsigned long long>& out,
                      cudaStream_t s) {
  if (out.n < count) out.alloc(count);
  if (count == 0) return 0;
  DevBuf<unsigned long long> nsel(1);
  size_t tmp = 0;
  AGPM_CUDA(cub::DeviceSelect::Unique(nullptr, tmp, keys.p, out.p, nsel.p, (int64_t)count, s));
  DevBuf<unsigned char> t(tmp + 16);
  AGPM_CUDA(cub::DeviceSelect::Unique(t.p, tmp, keys.p, out.p, nsel.p, (int64_t)count, s));
  unsigned long long u = 0, last = 0;
  AGPM_CUDA(cudaMemcpyAsync(&u, nsel.p, 8, cudaMemcpyDeviceToHost, s));
  AGPM_CUDA(cudaStreamSynchronize(s));
  if (u) {
    AGPM_CUDA(cudaMemcpyAsync(&last, out.p + u - 1, 8, cudaMemcpyDeviceToHost, s));
    AGPM_CUDA(cudaStreamSynchronize(s));
    if (last == kLoop) --u;
  }
  return u;
}

// rank of (degree, id) for every vertex -> new_id (relabel_by_degree order)
void degree_rank(const unsigned int* d_deg, uint32_t n, DevBuf<uint32_t>& new_id, int sm, cudaStream_t s) {
  DevBuf<unsigned int> deg_alt(n);
  DevBuf<uint32_t> ids(n), ids_alt(n);
  iota_kernel<<<grid_for(n, sm), 256, 0, s>>>(n, ids.p);
  count_launch();
  DevBuf<unsigned int> deg_copy(n);
  AGPM_CUDA(cudaMemcpyAsync(deg_copy.p, d_deg, 4ull * n, cudaMemcpyDeviceToDevice, s));
  cub::DoubleBuffer<unsigned int> dk(deg_copy.p, deg_alt.p);
  cub::DoubleBuffer<uint32_t> dv(ids.p, ids_alt.p);
  size_t tmp = 0;
  AGPM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, dk, dv, (int64_t)n, 0, 32, s));
  DevBuf<unsigned char> t(tmp + 16);
  // LSD radix sort is stable: equal degrees keep ascending ids
  AGPM_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, dk, dv, (int64_t)n, 0, 32, s));
  new_id.alloc(n);
  invert_kernel<<<grid_for(n, sm), 256, 0, s>>>(dv.Current(), n, new_id.p);
  count_launch();
  AGPM_CUDA(cudaGetLastError());
  AGPM_CUDA(cudaStreamSynchronize(s));
}

// Sorted arc keys (u<<32|v, u ascending then v ascending) -> a device view.
// Takes ownership of `arcs` (it becomes seed_arcs).
agpm_graph* view_from_sorted_arcs(DevBuf<unsigned long long>& arcs, uint64_t count, uint32_t n,
                                  uint64_t edge_count, bool oriented, int sm, cudaStream_t s) {
  auto* g = new agpm_graph();
  try {
    g->device = ctx_for_current_device().device;
    g->n = n;
    g->edge_count = edge_count;
    g->oriented = oriented;
    g->plain = true;
    g->loop_free = true;  // ingest drops self-loops (their keys sort last and are cut)
    g->nbr_len = count;
    g->arcs = count;
    g->nbr = alloc_nbr(count, s);
    DevBuf<unsigned long long> first(n ? n : 1), last(n ? n : 1), begin((size_t)n + 1);
    AGPM_CUDA(cudaMemsetAsync(first.p, 0, 8ull * first.n, s));
    AGPM_CUDA(cudaMemsetAsync(last.p, 0, 8ull * last.n, s));
    if (count) {
      bounds_kernel<<<grid_for(count, sm), 256, 0, s>>>(arcs.p, count, first.p, last.p, g->nbr);
      count_launch();
    }
    AGPM_CUDA(cudaMemsetAsync(begin.p, 0, 8, s));
    unsigned long long maxd = 0;
    if (n) {
      // deg into `first` is unsafe (aliasing); reuse `last` as the degree array
      deg_from_bounds_kernel<<<grid_for(n, sm), 256, 0, s>>>(first.p, last.p, n, last.p);
      count_launch();
      AGPM_CUDA(cudaGetLastError());
      DevBuf<unsigned long long> red(1);
      size_t t1 = 0, t2 = 0;
      AGPM_CUDA(cub::DeviceScan::InclusiveSum(nullptr, t1, last.p, begin.p + 1, (int64_t)n, s));
      AGPM_CUDA(cub::DeviceReduce::Max(nullptr, t2, last.p, red.p, (int64_t)n, s));
      DevBuf<unsigned char> t(std::max(t1, t2) + 16);
      AGPM_CUDA(cub::DeviceScan::InclusiveSum(t.p, t1, last.p, begin.p + 1, (int64_t)n, s));
      AGPM_CUDA(cub::DeviceReduce::Max(t.p, t2, last.p, red.p, (int64_t)n, s));
      AGPM_CUDA(cudaMemcpyAsync(&maxd, red.p, 8, cudaMemcpyDeviceToHost, s));
      AGPM_CUDA(dev_malloc(&g->vtx, sizeof(VtxInfo) * (size_t)n));
      vtx_from_bounds_kernel<<<grid_for(n, sm), 256, 0, s>>>(begin.p, g->nbr, n, g->vtx);
      count_launch();
      AGPM_CUDA(cudaGetLastError());
      AGPM_CUDA(cudaStreamSynchronize(s));
    } else {
      AGPM_CUDA(dev_malloc(&g->vtx, sizeof(VtxInfo)));
    }
    g->max_degree = maxd;
    if (count) {
      g->seed_arcs = arcs.take();
    } else {
      AGPM_CUDA(dev_malloc(&g->seed_arcs, 8));
    }
    g->bytes = sizeof(VtxInfo) * (uint64_t)n + 4ull * g->nbr_len + 8ull * g->arcs;
    return g;
  } catch (...) {
    dev_free(g->vtx);
    dev_free(g->nbr);
    dev_free(g->seed_arcs);
    delete g;
    throw;
  }
}

// Unsorted normalised edge keys (loops = kLoop) -> undirected device view,
// optionally degree-relabelled (host twins: graph_from_edges [+ relabel_by_degree]).
agpm_graph* build_from_edge_keys(DevBuf<unsigned long long>& keys, uint64_t count, uint32_t n, bool relabel,
                                 cudaStream_t s) {
  const int sm = ctx_for_current_device().sm_count;
  DevBuf<unsigned long long> alt;
  sort_keys(keys, alt, count, 64, s);
  // unique into the sort's spare buffer
  uint64_t m = unique_edges(keys, count, alt, s);
  keys.release();
  DevBuf<uint32_t> new_id;
  if (relabel && n) {
    DevBuf<unsigned int> deg(n);
    AGPM_CUDA(cudaMemsetAsync(deg.p, 0, 4ull * n, s));
    if (m) {
      degree_kernel<<<grid_for(m, sm), 256, 0, s>>>(alt.p, m, deg.p);
      count_launch();
      AGPM_CUDA(cudaGetLastError());
    }
    degree_rank(deg.p, n, new_id, sm, s);
  }
  DevBuf<unsigned long long> arcs(2 * m);
  if (m) {
    expand_kernel<<<grid_for(m, sm), 256, 0, s>>>(alt.p, m, new_id.p, arcs.p);
    count_launch();
    AGPM_CUDA(cudaGetLastError());
    AGPM_CUDA(cudaStreamSynchronize(s));
  }
  alt.release();
  new_id.release();
  DevBuf<unsigned long long> arcs_alt;
  sort_keys(arcs, arcs_alt, 2 * m, 32 + bits_for(n ? n - 1 : 0), s);
  arcs_alt.release();
  return view_from_sorted_arcs(arcs, 2 * m, n, m, false, sm, s);
}

}  // namespace
}  // namespace agpm_b200

using namespace agpm_b200;

extern "C" {

int agpm_gen_rmat_device(uint32_t scale, uint32_t edge_factor, double a, double b, double c, uint64_t seed,
                         int relabel, void* stream, agpm_graph** out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("null argument");
    if (scale < 1 || scale > 31) throw std::invalid_argument("rmat scale must be in [1,31]");
    DeviceCtx& ctx = ctx_for_current_device();
    cudaStream_t s = pick_stream(stream);
    const uint64_t m = static_cast<uint64_t>(edge_factor) << scale;
    DevBuf<unsigned long long> keys(m);
    if (m) {
      rmat_kernel<<<grid_for(m, ctx.sm_count), 256, 0, s>>>(scale, a, a + b, a + b + c, seed, m, keys.p);
      count_launch();
      AGPM_CUDA(cudaGetLastError());
    }
    *out = build_from_edge_keys(keys, m, 1u << scale, relabel != 0, s);
  });
}

int agpm_gen_er_fast_device(uint32_t n, uint64_t target_edges, uint64_t seed, uint32_t planted_k,
                            uint32_t planted_count, int relabel, void* stream, agpm_graph** out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("null argument");
    if (n < 2) throw std::invalid_argument("er_fast needs n >= 2");
    if (planted_k >= 2 && planted_k > n) throw std::invalid_argument("planted clique larger than the graph");
    DeviceCtx& ctx = ctx_for_current_device();
    cudaStream_t s = pick_stream(stream);
    // planted cliques: a handful of host draws (host_graph.cpp gen_er_fast)
    std::vector<unsigned long long> planted;
    if (planted_k >= 2) {
      for (uint32_t c = 0; c < planted_count; ++c) {
        CounterRng rng(seed, 0x706c616e74ull, c);
        std::vector<uint32_t> vs;
        while (vs.size() < planted_k) {
          auto v = static_cast<uint32_t>(rng.next_below(n));
          if (std::find(vs.begin(), vs.end(), v) == vs.end()) vs.push_back(v);
        }
        for (uint32_t x = 0; x < planted_k; ++x)
          for (uint32_t y = x + 1; y < planted_k; ++y)
            planted.push_back((static_cast<unsigned long long>(std::min(vs[x], vs[y])) << 32) |
                              std::max(vs[x], vs[y]));
      }
    }
    const uint64_t total = target_edges + planted.size();
    DevBuf<unsigned long long> keys(total);
    if (target_edges) {
      er_kernel<<<grid_for(target_edges, ctx.sm_count), 256, 0, s>>>(n, seed, target_edges, keys.p);
      count_launch();
      AGPM_CUDA(cudaGetLastError());
    }
    if (!planted.empty())
      AGPM_CUDA(cudaMemcpyAsync(keys.p + target_edges, planted.data(), 8 * planted.size(), cudaMemcpyHostToDevice, s));
    AGPM_CUDA(cudaStreamSynchronize(s));
    *out = build_from_edge_keys(keys, total, n, relabel != 0, s);
  });
}

int agpm_graph_from_edges_device(const uint32_t* pairs, uint64_t count, uint32_t min_vertex_count, int relabel,
                                 void* stream, agpm_graph** out) {
  return guarded([&] {
    if (!out || (count && !pairs)) throw std::invalid_argument("null argument");
    DeviceCtx& ctx = ctx_for_current_device();
    cudaStream_t s = pick_stream(stream);
    DevBuf<uint32_t> d_pairs(2 * count);
    DevBuf<unsigned long long> keys(count);
    DevBuf<unsigned int> max_id(1);
    AGPM_CUDA(cudaMemsetAsync(max_id.p, 0, 4, s));
    unsigned int mx = 0;
    if (count) {
      AGPM_CUDA(cudaMemcpyAsync(d_pairs.p, pairs, 8ull * count, cudaMemcpyHostToDevice, s));
      pairs_kernel<<<grid_for(count, ctx.sm_count), 256, 0, s>>>(d_pairs.p, count, keys.p, max_id.p);
      count_launch();
      AGPM_CUDA(cudaGetLastError());
      AGPM_CUDA(cudaMemcpyAsync(&mx, max_id.p, 4, cudaMemcpyDeviceToHost, s));
    }
    AGPM_CUDA(cudaStreamSynchronize(s));
    d_pairs.release();
    // csr_graph.cpp:46-72: n = max(min_vertex_count, max id + 1) (self-loops count)
    uint64_t n64 = min_vertex_count;
    if (count) n64 = std::max<uint64_t>(n64, (uint64_t)mx + 1);
    if (n64 > UINT32_MAX) throw std::invalid_argument("vertex count out of range");
    *out = build_from_edge_keys(keys, count, (uint32_t)n64, relabel != 0, s);
  });
}

int agpm_graph_relabel_device(const agpm_graph* g, void* stream, agpm_graph** out) {
  return guarded([&] {
    if (!g || !out) throw std::invalid_argument("null argument");
    if (g->oriented || !g->plain || g->arcs != g->nbr_len)
      throw std::invalid_argument("device relabel needs a plain undirected view");
    DeviceCtx& ctx = ctx_for_current_device();
    cudaStream_t s = pick_stream(stream);
    const uint32_t n = g->n;
    DevBuf<uint32_t> new_id;
    if (n) {
      DevBuf<unsigned int> deg(n);
      view_degree_kernel<<<grid_for(n, ctx.sm_count), 256, 0, s>>>(g->vtx, n, deg.p);
      count_launch();
      degree_rank(deg.p, n, new_id, ctx.sm_count, s);
    }
    DevBuf<unsigned long long> arcs(g->arcs);
    if (g->arcs) {
      remap_arcs_kernel<<<grid_for(g->arcs, ctx.sm_count), 256, 0, s>>>(g->seed_arcs, g->arcs, new_id.p, arcs.p);
      count_launch();
      AGPM_CUDA(cudaGetLastError());
    }
    new_id.release();
    DevBuf<unsigned long long> alt;
    sort_keys(arcs, alt, g->arcs, 32 + bits_for(n ? n - 1 : 0), s);
    alt.release();
    *out = view_from_sorted_arcs(arcs, g->arcs, n, g->edge_count, false, ctx.sm_count, s);
  });
}

int agpm_graph_orient_device(const agpm_graph* g, void* stream, agpm_graph** out) {
  return guarded([&] {
    if (!g || !out) throw std::invalid_argument("null argument");
    if (g->oriented || !g->plain || g->arcs != g->nbr_len)
      throw std::invalid_argument("device orientation needs a plain undirected view");
    DeviceCtx& ctx = ctx_for_current_device();
    cudaStream_t s = pick_stream(stream);
    // selecting from the sorted arc keys keeps them sorted: no re-sort
    DevBuf<unsigned long long> arcs(g->arcs), nsel(1);
    uint64_t kept = 0;
    if (g->arcs) {
      size_t tmp = 0;
      OrientKeep keep{g->vtx};
      AGPM_CUDA(cub::DeviceSelect::If(nullptr, tmp, g->seed_arcs, arcs.p, nsel.p, (int64_t)g->arcs, keep, s));
      DevBuf<unsigned char> t(tmp + 16);
      AGPM_CUDA(cub::DeviceSelect::If(t.p, tmp, g->seed_arcs, arcs.p, nsel.p, (int64_t)g->arcs, keep, s));
      unsigned long long k = 0;
      AGPM_CUDA(cudaMemcpyAsync(&k, nsel.p, 8, cudaMemcpyDeviceToHost, s));
      AGPM_CUDA(cudaStreamSynchronize(s));
      kept = k;
    }
    *out = view_from_sorted_arcs(arcs, kept, g->n, g->edge_count, true, ctx.sm_count, s);
  });
}

}  // extern "C"
