// Dense/sparse degree-threshold region split (builder-
// defined — the reference has no implementation).
//
// Definition: V_s = {v : deg(v) < tau}, V_d = the rest.
//   C_sparse = #matches with at least one vertex in V_s, counted EXACTLY;
//   C_dense  = #matches inside G[V_d], estimated (online NS to eps@delta,
//              repeated colour-GS, or exact);
//   estimate = C_sparse + C_dense.
// On a degree-relabelled graph (id = rank of (degree, id)) V_s is the id prefix
// [0, tau_id). When the plan's symmetry constraints force matching position 0
// to hold the smallest id of every match (cliques, 4-cycle, ...; checked on
// the constraint closure) — or the view is a degree-oriented clique DAG — a
// match touches V_s iff its root v0 < tau_id, so C_sparse is the exact count
// restricted to roots below tau_id; otherwise C_sparse = exact(G) - exact(G[V_d]).
// Parity is pinned by composition: C_sparse + exact(G[V_d]) == exact(G).
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "device.cuh"
#include "rng.cuh"

namespace agpm_b200 {

namespace {

constexpr unsigned FULLM = 0xffffffffu;

// #vertices with degree < tau, and whether degrees are non-decreasing in id order
__global__ void degree_scan_kernel(const VtxInfo* __restrict__ vtx, uint32_t n, uint32_t tau,
                                   unsigned long long* __restrict__ below, unsigned int* __restrict__ unsorted) {
  unsigned long long cnt = 0;
  unsigned bad = 0;
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < n; u += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t d = vtx[u].deg;
    cnt += d < tau;
    if (u + 1 < n && vtx[u + 1].deg < d) bad = 1;
  }
  for (int o = 16; o > 0; o >>= 1) {
    cnt += __shfl_xor_sync(FULLM, cnt, o);
    bad |= __shfl_xor_sync(FULLM, bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (cnt) atomicAdd(below, cnt);
    if (bad) atomicOr(unsorted, 1u);
  }
}

// G[V_d]: keep arc (u, v) iff u >= lo and v >= lo (ids unchanged)
__global__ void induced_count_kernel(const VtxInfo* __restrict__ vtx, const uint32_t* __restrict__ nbr, uint32_t n,
                                     uint32_t lo, unsigned long long* __restrict__ kept) {
  const int lane = threadIdx.x & 31;
  const uint64_t w0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t u = w0; u < n; u += nw) {
    const VtxInfo vi = vtx[u];
    uint32_t k = 0;
    if (u >= lo)
      for (uint32_t c0 = 0; c0 < vi.deg; c0 += 32) {
        const bool keep = c0 + lane < vi.deg && nbr[vi.begin + c0 + lane] >= lo;
        k += __popc(__ballot_sync(FULLM, keep));
      }
    if (lane == 0) kept[u] = k;
  }
}

__global__ void induced_fill_kernel(const VtxInfo* __restrict__ vtx, const uint32_t* __restrict__ nbr, uint32_t n,
                                    uint32_t lo, const unsigned long long* __restrict__ offs, uint32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const uint64_t w0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t u = w0; u < n; u += nw) {
    if (u < lo) continue;
    const VtxInfo vi = vtx[u];
    unsigned long long at = offs[u];
    for (uint32_t c0 = 0; c0 < vi.deg; c0 += 32) {
      const bool valid = c0 + lane < vi.deg;
      const uint32_t x = valid ? nbr[vi.begin + c0 + lane] : 0;
      const bool keep = valid && x >= lo;
      const unsigned bk = __ballot_sync(FULLM, keep);
      if (keep) out[at + __popc(bk & ((1u << lane) - 1u))] = x;
      at += __popc(bk);
    }
  }
}

unsigned grid(uint64_t warps_work) {
  DeviceCtx& ctx = ctx_for_current_device();
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((warps_work + 7) / 8, (uint64_t)ctx.sm_count * 16));
}

// does the constraint closure put order[0] below every other pattern vertex?
bool root_is_minimum(const agpm_plan* p) {
  const int k = p->k;
  bool less[AGPM_MAX_K][AGPM_MAX_K] = {};
  for (int i = 0; i < p->n_constraints; ++i) less[p->constraints[i][0]][p->constraints[i][1]] = true;
  for (int m = 0; m < k; ++m)
    for (int a = 0; a < k; ++a)
      for (int b = 0; b < k; ++b)
        if (less[a][m] && less[m][b]) less[a][b] = true;
  const int r = p->order[0];
  for (int x = 0; x < k; ++x)
    if (x != r && !less[r][x]) return false;
  return true;
}

}  // namespace

agpm_graph* induced_suffix_device(const agpm_graph* g, uint32_t lo, cudaStream_t s) {
  DeviceCtx& ctx = ctx_for_current_device();
  const uint32_t n = g->n;
  unsigned long long* offs = nullptr;
  AGPM_CUDA(dev_malloc(&offs, 8ull * ((size_t)n + 1)));
  AGPM_CUDA(cudaMemsetAsync(offs + n, 0, 8, s));
  if (n) {
    induced_count_kernel<<<grid(n), 256, 0, s>>>(g->vtx, g->nbr, n, lo, offs);
    count_launch();
    AGPM_CUDA(cudaGetLastError());
  }
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, offs, offs, (int64_t)n + 1, s);
  void* tmp = ctx.get(7, tb + 16);
  AGPM_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, offs, offs, (int64_t)n + 1, s));
  unsigned long long kept = 0;
  AGPM_CUDA(cudaMemcpyAsync(&kept, offs + n, 8, cudaMemcpyDeviceToHost, s));
  AGPM_CUDA(cudaStreamSynchronize(s));
  auto* out = new agpm_graph();
  out->device = g->device;
  out->n = n;
  out->oriented = g->oriented;
  out->edge_count = g->oriented ? kept : kept / 2;
  out->nbr_len = kept;
  out->plain = true;
  out->nbr = alloc_nbr(kept, s);
  if (n) {
    induced_fill_kernel<<<grid(n), 256, 0, s>>>(g->vtx, g->nbr, n, lo, offs, out->nbr);
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

int agpm_induced_suffix(agpm_graph* g, uint32_t min_vertex, agpm_graph** out, void* stream) {
  return guarded([&] {
    if (!g || !out) throw std::invalid_argument("null argument");
    *out = induced_suffix_device(g, min_vertex, pick_stream(stream));
  });
}

int agpm_region_split(agpm_graph* g, const agpm_plan* plan, uint32_t tau_degree, int dense_method, double eps,
                      double delta, uint64_t seed, uint32_t colors, uint32_t repeats, uint64_t max_samples,
                      agpm_region_result* out, void* stream) {
  return guarded([&] {
    if (!g || !plan || !out) throw std::invalid_argument("null argument");
    if (dense_method < 0 || dense_method > 2) throw std::invalid_argument("dense method: 0 NS, 1 colour GS, 2 exact");
    cudaStream_t s = pick_stream(stream);
    DeviceCtx& ctx = ctx_for_current_device();
    std::memset(out, 0, sizeof(*out));
    auto t0 = std::chrono::steady_clock::now();
    auto* scratch = static_cast<unsigned long long*>(ctx.get(3, 64));
    AGPM_CUDA(cudaMemsetAsync(scratch, 0, 16, s));
    if (g->n) {
      degree_scan_kernel<<<grid(g->n / 32 + 1), 256, 0, s>>>(g->vtx, g->n, tau_degree, scratch,
                                                             reinterpret_cast<unsigned int*>(scratch + 1));
      count_launch();
      AGPM_CUDA(cudaGetLastError());
    }
    unsigned long long h[2] = {0, 0};
    AGPM_CUDA(cudaMemcpyAsync(h, scratch, 16, cudaMemcpyDeviceToHost, s));
    AGPM_CUDA(cudaStreamSynchronize(s));
    // an oriented DAG's out-degrees are not the degrees the split is defined on:
    // there `tau` is the id threshold itself (the symmetric view's tau_id)
    if (!g->oriented && h[1])
      throw std::invalid_argument("region split needs a degree-relabelled graph (degrees ascending with id)");
    const uint32_t tau_id = g->oriented ? std::min(tau_degree, g->n) : static_cast<uint32_t>(h[0]);
    out->tau_id = tau_id;
    out->sparse_vertices = tau_id;
    out->dense_vertices = g->n - tau_id;
    const bool clique = plan->n_edges == plan->k * (plan->k - 1) / 2;
    out->rooted = (g->oriented && clique) || root_is_minimum(plan);
    agpm_graph* dense = induced_suffix_device(g, tau_id, s);
    out->dense_edges = dense->edge_count;
    try {
      if (out->rooted && plan_is_plain_4cycle(plan) && g->plain && !g->oriented) {
        // 4-cycles: pair aggregation instead of the wedge-by-wedge DFS through hubs
        out->c_sparse = cycle4_sparse_count(g, tau_id, s);
      } else if (out->rooted) {
        out->c_sparse = exact_count_device(g, plan, s, tau_id);
      } else {
        out->c_sparse = exact_count_device(g, plan, s, 0xffffffffu) - exact_count_device(dense, plan, s, 0xffffffffu);
      }
      auto t1 = std::chrono::steady_clock::now();
      out->sparse_seconds = std::chrono::duration<double>(t1 - t0).count();
      if (dense->edge_count == 0) {
        out->c_dense = 0.0;
        out->dense_exact = 1;
      } else if (dense_method == 2) {
        out->c_dense = static_cast<double>(exact_count_device(dense, plan, s, 0xffffffffu));
        out->dense_exact = 1;
      } else if (dense_method == 1) {
        // repeated colourings, each an unbiased coarse sample c^(k-1) x raw
        // (gs_engine.cpp:42-75), run under the online detector to eps@delta
        // (Appendix C.2) with `repeats` as the cap on colourings
        if (agpm_gs_online(dense, plan, colors, eps, delta, std::max<uint32_t>(2, repeats), seed, &out->dense_ns, s) !=
            AGPM_OK)
          throw std::runtime_error(agpm_last_error());
        out->c_dense = out->dense_ns.report.mu;
        out->dense_epsilon_hat = out->dense_ns.report.epsilon_hat;
      } else {
        agpm_online_policy pol{1000, max_samples ? max_samples : 1000000000ull, 0};
        if (agpm_ns_online(dense, plan, eps, delta, &pol, seed, &out->dense_ns, s) != AGPM_OK)
          throw std::runtime_error(agpm_last_error());
        out->c_dense = out->dense_ns.report.mu;
        out->dense_epsilon_hat = out->dense_ns.report.epsilon_hat;
      }
      out->dense_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
    } catch (...) {
      agpm_graph_free(dense);
      throw;
    }
    agpm_graph_free(dense);
    out->estimate = static_cast<double>(out->c_sparse) + out->c_dense;
  });
}

int agpm_gs_online(agpm_graph* g, const agpm_plan* plan, uint32_t colors, double eps, double delta,
                   uint64_t max_colorings, uint64_t seed, agpm_online_result* out, void* stream) {
  // Colour-sparsified GS run to a relative error bound:
  // colouring i (colours from derive_key(seed, i, 0)) gives the unbiased coarse
  // sample X_i = c^(k-1) x raw_i (gs_engine.cpp:42-75); the X_i are i.i.d., so
  // the NS online detector applies unchanged — accumulate (n, hits, sum, sum of
  // squares) and stop at the first i >= 2 with eps_hat <= eps (stats.cpp:57-70),
  // or at max_colorings.
  return guarded([&] {
    if (!g || !plan || !out) throw std::invalid_argument("null argument");
    if (!(eps > 0.0) || !(eps < 1.0)) throw std::invalid_argument("error bound must be inside (0,1)");
    if (!(delta > 0.0) || !(delta < 1.0)) throw std::invalid_argument("delta must be inside (0,1)");
    if (colors < 1) throw std::invalid_argument("color count must be >= 1");
    if (max_colorings < 1) throw std::invalid_argument("need at least one colouring");
    cudaStream_t s = pick_stream(stream);
    std::memset(out, 0, sizeof(*out));
    agpm_accumulator acc{0, 0, 0.0, 0.0};
    agpm_report rep{};
    const auto t0 = std::chrono::steady_clock::now();
    for (uint64_t i = 0; i < max_colorings; ++i) {
      agpm_gs_result gr{};
      if (agpm_gs_estimate(g, plan, 1, 1.0, colors, derive_key(seed, i, 0), &gr, s) != AGPM_OK)
        throw std::runtime_error(agpm_last_error());
      acc.n += 1;
      acc.hits += gr.raw_count ? 1 : 0;
      acc.sum += gr.estimate;
      acc.squared_sum += gr.estimate * gr.estimate;
      if (agpm_predicted_error(&acc, delta, &rep) != AGPM_OK) throw std::runtime_error(agpm_last_error());
      out->windows = i + 1;
      if (rep.epsilon_hat <= eps) {
        rep.converged = 1;
        break;
      }
    }
    out->report = rep;
    out->accumulator = acc;
    out->samples_launched = acc.n;
    out->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

}  // extern "C"
