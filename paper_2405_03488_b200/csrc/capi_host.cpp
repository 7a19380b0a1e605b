// C-ABI for host CSR graphs and generators (include/agpm_b200.h).
#include <atomic>
#include <cstring>

#include "common.hpp"
#include "host_graph.hpp"

using namespace agpm_b200;

namespace {
agpm_host_graph* wrap(HostGraph&& g) {
  auto* h = new agpm_host_graph();
  h->g = std::move(g);
  return h;
}
void need(const void* p) {
  if (!p) throw std::invalid_argument("null argument");
}
}  // namespace

uint64_t agpm_b200_next_generation() {
  static std::atomic<uint64_t> next{1};
  return next.fetch_add(1);
}

extern "C" {

int agpm_host_graph_generation(const agpm_host_graph* g, uint64_t* out) {
  return guarded([&] {
    need(g);
    need(out);
    *out = g->generation;
  });
}

int agpm_host_graph_from_edges(const uint32_t* edges, uint64_t n_edges, uint32_t min_n,
                               agpm_host_graph** out) {
  return guarded([&] {
    need(out);
    if (n_edges) need(edges);
    std::vector<std::pair<uint32_t, uint32_t>> e(n_edges);
    for (uint64_t i = 0; i < n_edges; ++i) e[i] = {edges[2 * i], edges[2 * i + 1]};
    *out = wrap(graph_from_edges(e, min_n));
  });
}

int agpm_host_graph_from_csr(uint32_t n, uint64_t edge_count, const uint64_t* offsets,
                             const uint32_t* neighbors, int oriented, agpm_host_graph** out) {
  return guarded([&] {
    need(out);
    need(offsets);
    HostGraph g;
    g.n = n;
    g.edge_count = edge_count;
    g.oriented = oriented != 0;
    g.offsets.assign(offsets, offsets + n + 1);
    if (g.offsets.back()) need(neighbors);
    g.neighbors.assign(neighbors, neighbors + g.offsets.back());
    *out = wrap(std::move(g));
  });
}

int agpm_host_graph_load(const char* path, agpm_host_graph** out) {
  return guarded([&] {
    need(path);
    need(out);
    *out = wrap(load_auto(path));
  });
}

int agpm_host_graph_write_binary(const agpm_host_graph* g, const char* path) {
  return guarded([&] {
    need(g);
    need(path);
    write_binary(g->g, path);
  });
}

int agpm_host_graph_info(const agpm_host_graph* g, uint32_t* n, uint64_t* edge_count, uint64_t* arcs,
                         int* oriented, uint64_t* max_degree) {
  return guarded([&] {
    need(g);
    if (n) *n = g->g.n;
    if (edge_count) *edge_count = g->g.edge_count;
    if (arcs) *arcs = g->g.offsets.back();
    if (oriented) *oriented = g->g.oriented;
    if (max_degree) *max_degree = g->g.max_degree();
  });
}

int agpm_host_graph_arrays(const agpm_host_graph* g, const uint64_t** offsets, const uint32_t** nbr) {
  return guarded([&] {
    need(g);
    if (offsets) *offsets = g->g.offsets.data();
    if (nbr) *nbr = g->g.neighbors.data();
  });
}

void agpm_host_graph_free(agpm_host_graph* g) {
  agpm_b200_unpin_host_graph(g);
  delete g;
}

int agpm_host_graph_relabel_by_degree(const agpm_host_graph* g, agpm_host_graph** out) {
  return guarded([&] {
    need(g);
    need(out);
    *out = wrap(relabel_by_degree(g->g));
  });
}

int agpm_host_graph_orient_by_degree(const agpm_host_graph* g, agpm_host_graph** out) {
  return guarded([&] {
    need(g);
    need(out);
    *out = wrap(orient_by_degree(g->g));
  });
}

int agpm_gen_er_pairs(uint32_t n, double p, uint64_t seed, agpm_host_graph** out) {
  return guarded([&] {
    need(out);
    *out = wrap(gen_er_pairs(n, p, seed));
  });
}

int agpm_gen_er_fast(uint32_t n, uint64_t target_edges, uint64_t seed, uint32_t planted_k,
                     uint32_t planted_count, agpm_host_graph** out) {
  return guarded([&] {
    need(out);
    *out = wrap(gen_er_fast(n, target_edges, seed, planted_k, planted_count));
  });
}

int agpm_gen_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c, uint64_t seed,
                  agpm_host_graph** out) {
  return guarded([&] {
    need(out);
    *out = wrap(gen_rmat(scale, edge_factor, a, b, c, seed));
  });
}

}  // extern "C"
