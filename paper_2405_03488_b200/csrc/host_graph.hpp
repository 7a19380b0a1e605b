// Host-side CSR graph: construction, binary I/O, degree relabelling and the
// deterministic generators used by the benchmark configs. Mirrors the data
// contract of agpm::CsrGraph (csr_graph.hpp:43-80): u64 offsets, u32 strictly
// ascending neighbour lists, no self-loops or duplicates, symmetric unless
// oriented. Construction is multi-threaded (the reference's from_edges is a
// single-thread sort, csr_graph.cpp:46-72); the resulting arrays are identical.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

namespace agpm_b200 {

struct HostGraph {
  uint32_t n = 0;
  uint64_t edge_count = 0;  // undirected edges (== arcs when oriented)
  bool oriented = false;
  std::vector<uint64_t> offsets{0};
  std::vector<uint32_t> neighbors;

  uint64_t degree(uint32_t u) const { return offsets[u + 1] - offsets[u]; }
  uint64_t max_degree() const;
};

// CsrGraph::from_edges (csr_graph.cpp:46-72); `pairs` is consumed.
HostGraph graph_from_edges(std::vector<std::pair<uint32_t, uint32_t>>& pairs,
                           uint32_t min_vertex_count);

// Binary "AGPM" v1 format (csr_graph.cpp:109-160) and the text edge list
// fallback of load_graph_auto (csr_graph.cpp:74-93, 162-170).
void write_binary(const HostGraph& g, const std::string& path);
HostGraph load_auto(const std::string& path);

// id := rank of (degree, id), neighbour lists re-sorted.
HostGraph relabel_by_degree(const HostGraph& g);
// orient_by_degree (csr_graph.cpp:172-188)
HostGraph orient_by_degree(const HostGraph& g);

// Generators (see agpm_b200.h)
HostGraph gen_er_pairs(uint32_t n, double p, uint64_t seed);
HostGraph gen_er_fast(uint32_t n, uint64_t target_edges, uint64_t seed, uint32_t planted_k,
                      uint32_t planted_count);
HostGraph gen_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                   uint64_t seed);

}  // namespace agpm_b200

uint64_t agpm_b200_next_generation();

// C-ABI opaque handle (agpm_b200.h)
struct agpm_host_graph {
  agpm_b200::HostGraph g;
  bool pinned = false;
  // process-unique id (never reused): keys device-mirror caches so a freed
  // graph's recycled addresses can never alias a new graph's (include/agpm/agpm.hpp)
  uint64_t generation = agpm_b200_next_generation();
};
void agpm_b200_unpin_host_graph(agpm_host_graph* g);
