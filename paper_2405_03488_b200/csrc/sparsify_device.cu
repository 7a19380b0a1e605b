// Graph sparsification on the device:
//   colour split   ColoredCsr::color_vertices + build_splits (colored_csr.cpp:14-54)
//   Bernoulli      bernoulli_sparsify (csr_graph.cpp:190-213)
//   GS estimate    gs_estimate (gs_engine.cpp:42-75)
// Decisions are the reference's stateless hashes (rng.hpp:60-70), so the
// sparsified graphs are identical arc for arc; both passes are warp-per-vertex
// stable partitions / compactions with ballot prefix sums.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>
#include <cstring>
#include <chrono>
#include <cmath>
#include <stdexcept>

#include "device.cuh"
#include "rng.cuh"

namespace agpm_b200 {

namespace {

constexpr unsigned FULLM = 0xffffffffu;

__global__ void colors_kernel(uint32_t n, uint64_t seed, uint32_t c, uint32_t* __restrict__ colors) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x)
    colors[v] = vertex_color_decision(seed, (uint32_t)v, c);  // colored_csr.cpp:48-54
}

// warp per vertex: [same colour (ascending) | rest (ascending)] = std::stable_partition
__global__ void color_split_kernel(const VtxInfo* __restrict__ vtx, const uint32_t* __restrict__ nbr, uint32_t n,
                                   const uint32_t* __restrict__ colors, uint32_t* __restrict__ out,
                                   unsigned long long* __restrict__ begin, unsigned long long* __restrict__ split,
                                   unsigned long long* __restrict__ same_total) {
  const int lane = threadIdx.x & 31;
  const uint64_t w0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long same_acc = 0;
  for (uint64_t u = w0; u < n; u += nw) {
    const VtxInfo vi = vtx[u];
    const uint32_t cu = colors[u];
    uint32_t nsame = 0;
    for (uint32_t c0 = 0; c0 < vi.deg; c0 += 32) {
      const bool valid = c0 + lane < vi.deg;
      const bool same = valid && colors[nbr[vi.begin + c0 + lane]] == cu;
      nsame += __popc(__ballot_sync(FULLM, same));
    }
    uint32_t a = 0, b = nsame;
    for (uint32_t c0 = 0; c0 < vi.deg; c0 += 32) {
      const bool valid = c0 + lane < vi.deg;
      const uint32_t x = valid ? nbr[vi.begin + c0 + lane] : 0;
      const bool same = valid && colors[x] == cu;
      const unsigned bs = __ballot_sync(FULLM, same), bo = __ballot_sync(FULLM, valid && !same);
      const unsigned below = (1u << lane) - 1u;
      if (same) out[vi.begin + a + __popc(bs & below)] = x;
      else if (valid) out[vi.begin + b + __popc(bo & below)] = x;
      a += __popc(bs);
      b += __popc(bo);
    }
    if (lane == 0) {
      begin[u] = vi.begin;
      split[u] = vi.begin + nsame;
    }
    same_acc += nsame;
  }
  if (lane == 0 && same_acc) atomicAdd(same_total, same_acc);
}

// warp per vertex: kept-arc counts, then compaction (edge_keep_decision, rng.hpp:60-65)
__global__ void bern_count_kernel(const VtxInfo* __restrict__ vtx, const uint32_t* __restrict__ nbr, uint32_t n,
                                  uint64_t seed, double p, unsigned long long* __restrict__ kept) {
  const int lane = threadIdx.x & 31;
  const uint64_t w0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t u = w0; u < n; u += nw) {
    const VtxInfo vi = vtx[u];
    uint32_t k = 0;
    for (uint32_t c0 = 0; c0 < vi.deg; c0 += 32) {
      const bool valid = c0 + lane < vi.deg;
      const bool keep = valid && edge_keep_decision(seed, (uint32_t)u, nbr[vi.begin + c0 + lane], p);
      k += __popc(__ballot_sync(FULLM, keep));
    }
    if (lane == 0) kept[u] = k;
  }
}

__global__ void bern_fill_kernel(const VtxInfo* __restrict__ vtx, const uint32_t* __restrict__ nbr, uint32_t n,
                                 uint64_t seed, double p, const unsigned long long* __restrict__ offs,
                                 uint32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const uint64_t w0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t u = w0; u < n; u += nw) {
    const VtxInfo vi = vtx[u];
    unsigned long long at = offs[u];
    for (uint32_t c0 = 0; c0 < vi.deg; c0 += 32) {
      const bool valid = c0 + lane < vi.deg;
      const uint32_t x = valid ? nbr[vi.begin + c0 + lane] : 0;
      const bool keep = valid && edge_keep_decision(seed, (uint32_t)u, x, p);
      const unsigned bk = __ballot_sync(FULLM, keep);
      if (keep) out[at + __popc(bk & ((1u << lane) - 1u))] = x;
      at += __popc(bk);
    }
  }
}

unsigned grid_for(uint64_t items_per_warp_n) {
  DeviceCtx& ctx = ctx_for_current_device();
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((items_per_warp_n + 7) / 8, (uint64_t)ctx.sm_count * 16));
}

}  // namespace

// colour split of g with colours from the seed (colour_vertices) or, with
// explicit != null, from that host array (with_colors)
agpm_graph* color_split_impl(const agpm_graph* g, uint32_t c, uint64_t seed, const uint32_t* explicit_host,
                             uint32_t* colors_host, uint64_t* same_edges, cudaStream_t s) {
  if (c < 1) throw std::invalid_argument("color count must be >= 1");
  if (g->oriented) throw std::invalid_argument("colour sparsification needs the symmetric graph");
  DeviceCtx& ctx = ctx_for_current_device();
  const uint32_t n = g->n;
  auto* out = new agpm_graph();
  out->device = g->device;
  out->n = n;
  out->nbr_len = g->nbr_len;
  out->plain = false;
  out->oriented = false;
  uint32_t* colors = nullptr;
  unsigned long long *begin = nullptr, *split = nullptr;
  AGPM_CUDA(dev_malloc(&colors, 4ull * (n ? n : 1)));
  AGPM_CUDA(dev_malloc(&begin, 8ull * (n ? n : 1)));
  AGPM_CUDA(dev_malloc(&split, 8ull * (n ? n : 1)));
  out->nbr = alloc_nbr(g->nbr_len, s);
  auto* tot = static_cast<unsigned long long*>(ctx.get(3, 64));
  AGPM_CUDA(cudaMemsetAsync(tot, 0, 8, s));
  if (n) {
    if (explicit_host) {
      AGPM_CUDA(cudaMemcpyAsync(colors, explicit_host, 4ull * n, cudaMemcpyHostToDevice, s));
    } else {
      colors_kernel<<<grid_for((n + 31) / 32 * 8), 256, 0, s>>>(n, seed, c, colors);
    }
    color_split_kernel<<<grid_for(n), 256, 0, s>>>(g->vtx, g->nbr, n, colors, out->nbr, begin, split, tot);
    count_launch(explicit_host ? 1 : 2);
    AGPM_CUDA(cudaGetLastError());
  }
  unsigned long long same = 0;
  AGPM_CUDA(cudaMemcpyAsync(&same, tot, 8, cudaMemcpyDeviceToHost, s));
  if (colors_host && n) AGPM_CUDA(cudaMemcpyAsync(colors_host, colors, 4ull * n, cudaMemcpyDeviceToHost, s));
  AGPM_CUDA(cudaStreamSynchronize(s));
  out->edge_count = same / 2;  // same_color_edge_count (colored_csr.cpp:45)
  if (same_edges) *same_edges = same / 2;
  finalize_view(out, begin, split, s);
  AGPM_CUDA(dev_free(colors));
  AGPM_CUDA(dev_free(begin));
  AGPM_CUDA(dev_free(split));
  return out;
}

agpm_graph* color_split_device(const agpm_graph* g, uint32_t c, uint64_t seed, uint32_t* colors_host,
                               uint64_t* same_edges, cudaStream_t s) {
  return color_split_impl(g, c, seed, nullptr, colors_host, same_edges, s);
}

agpm_graph* bernoulli_device(const agpm_graph* g, double p, uint64_t seed, cudaStream_t s) {
  if (!(p > 0.0) || p > 1.0) throw std::invalid_argument("keep probability must be in (0,1]");
  DeviceCtx& ctx = ctx_for_current_device();
  const uint32_t n = g->n;
  unsigned long long* offs = nullptr;
  AGPM_CUDA(dev_malloc(&offs, 8ull * ((size_t)n + 1)));
  AGPM_CUDA(cudaMemsetAsync(offs + n, 0, 8, s));
  if (n) {
    bern_count_kernel<<<grid_for(n), 256, 0, s>>>(g->vtx, g->nbr, n, seed, p, offs);
    count_launch();
    AGPM_CUDA(cudaGetLastError());
  }
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, offs, offs, (int64_t)n + 1, s);
  void* tmp = ctx.get(7, tmp_bytes + 16);
  AGPM_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, offs, offs, (int64_t)n + 1, s));
  unsigned long long kept = 0;
  AGPM_CUDA(cudaMemcpyAsync(&kept, offs + n, 8, cudaMemcpyDeviceToHost, s));
  AGPM_CUDA(cudaStreamSynchronize(s));
  auto* out = new agpm_graph();
  out->device = g->device;
  out->n = n;
  out->edge_count = kept / 2;  // csr_graph.cpp:211
  out->nbr_len = kept;
  out->plain = true;
  out->nbr = alloc_nbr(kept, s);
  if (n) {
    bern_fill_kernel<<<grid_for(n), 256, 0, s>>>(g->vtx, g->nbr, n, seed, p, offs, out->nbr);
    count_launch();
    AGPM_CUDA(cudaGetLastError());
  }
  finalize_view(out, offs, nullptr, s);
  AGPM_CUDA(dev_free(offs));
  return out;
}

}  // namespace agpm_b200

using namespace agpm_b200;

extern "C" {

int agpm_color_split(agpm_graph* g, uint32_t colors, uint64_t seed, uint32_t* colors_out, uint64_t* same_edges,
                     agpm_graph** out, void* stream) {
  return guarded([&] {
    if (!g || !out) throw std::invalid_argument("null argument");
    *out = color_split_device(g, colors, seed, colors_out, same_edges, pick_stream(stream));
  });
}

int agpm_color_split_with_colors(agpm_graph* g, const uint32_t* colors, uint32_t color_count, uint64_t* same_edges,
                                 agpm_graph** out, void* stream) {
  // ColoredCsr::with_colors (colored_csr.cpp:14-46): an explicit assignment
  return guarded([&] {
    if (!g || !out || (g->n && !colors)) throw std::invalid_argument("null argument");
    for (uint32_t v = 0; v < g->n; ++v)
      if (colors[v] >= color_count) throw std::invalid_argument("color out of range");
    *out = color_split_impl(g, color_count, 0, colors, nullptr, same_edges, pick_stream(stream));
  });
}

int agpm_merge_colors(agpm_graph* g, const uint32_t* colors, uint32_t color_count, const uint32_t* group_map,
                      uint32_t map_len, uint32_t* coarse_out, uint64_t* same_edges, agpm_graph** out,
                      void* stream) {
  // ColoredCsr::merge_colors (colored_csr.cpp:56-88). Coarsening keeps each
  // list as [same-group neighbours ascending | the rest ascending] — exactly
  // the layout with_colors builds for the coarse colours on the original
  // (sorted) lists, so the merged view is the colour split of the coarse map.
  return guarded([&] {
    if (!g || !out || !group_map || (g->n && !colors)) throw std::invalid_argument("null argument");
    if (map_len != color_count) throw std::invalid_argument("group map must cover every color");
    uint32_t coarse_count = 0;
    for (uint32_t i = 0; i < map_len; ++i) coarse_count = std::max(coarse_count, group_map[i] + 1);
    std::vector<bool> seen(coarse_count, false);
    for (uint32_t i = 0; i < map_len; ++i) seen[group_map[i]] = true;
    for (bool b : seen)
      if (!b) throw std::invalid_argument("group map must be surjective onto a contiguous range");
    std::vector<uint32_t> coarse(g->n);
    for (uint32_t v = 0; v < g->n; ++v) {
      if (colors[v] >= color_count) throw std::invalid_argument("color out of range");
      coarse[v] = group_map[colors[v]];
    }
    if (coarse_out && g->n) std::memcpy(coarse_out, coarse.data(), 4ull * g->n);
    *out = color_split_impl(g, coarse_count, 0, coarse.data(), nullptr, same_edges, pick_stream(stream));
  });
}

int agpm_bernoulli_sparsify(agpm_graph* g, double keep_probability, uint64_t seed, agpm_graph** out,
                            void* stream) {
  return guarded([&] {
    if (!g || !out) throw std::invalid_argument("null argument");
    *out = bernoulli_device(g, keep_probability, seed, pick_stream(stream));
  });
}

int agpm_gs_estimate(agpm_graph* g, const agpm_plan* plan, int scheme, double keep_probability, uint32_t colors,
                     uint64_t seed, agpm_gs_result* out, void* stream) {
  // gs_estimate (gs_engine.cpp:42-75)
  return guarded([&] {
    if (!g || !plan || !out) throw std::invalid_argument("null argument");
    if (scheme == 0 && plan->induced)
      throw std::invalid_argument("edge sparsification supports edge-induced counting only; use the color scheme");
    if (scheme != 0 && scheme != 1) throw std::invalid_argument("scheme must be 0 (Bernoulli) or 1 (colour)");
    cudaStream_t s = pick_stream(stream);
    *out = agpm_gs_result{};
    auto t0 = std::chrono::steady_clock::now();
    agpm_graph* sp = scheme == 0 ? bernoulli_device(g, keep_probability, seed, s)
                                 : color_split_device(g, colors, seed, nullptr, nullptr, s);
    auto t1 = std::chrono::steady_clock::now();
    try {
      out->raw_count = exact_count_device(sp, plan, s);
    } catch (...) {
      agpm_graph_free(sp);
      throw;
    }
    auto t2 = std::chrono::steady_clock::now();
    agpm_graph_free(sp);
    out->scale = scheme == 0 ? std::pow(keep_probability, -plan->n_edges)
                             : std::pow(static_cast<double>(colors), plan->k - 1);
    out->estimate = static_cast<double>(out->raw_count) * out->scale;
    out->preprocess_seconds = std::chrono::duration<double>(t1 - t0).count();
    out->search_seconds = std::chrono::duration<double>(t2 - t1).count();
  });
}

int agpm_triangle_count(agpm_graph* g, uint64_t* count, void* stream) {
  // triangle_count (csr_graph.cpp:225-239): every triangle once
  return guarded([&] {
    if (!g || !count) throw std::invalid_argument("null argument");
    agpm_plan plan{};
    if (agpm_plan_compile("triangle", "", 0, 1, &plan) != AGPM_OK) throw std::runtime_error(agpm_last_error());
    *count = exact_count_device(g, &plan, pick_stream(stream));
  });
}

}  // extern "C"
