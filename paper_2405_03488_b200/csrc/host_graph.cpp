#include "host_graph.hpp"

#include <algorithm>
#include <cstring>
#include <fstream>
#include <numeric>
#include <sstream>
#include <stdexcept>
#include <thread>

#include "common.hpp"
#include "rng.cuh"

namespace agpm_b200 {

void parallel_for(uint64_t n, uint64_t grain, const std::function<void(uint64_t, uint64_t)>& body) {
  unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  uint64_t chunks = std::min<uint64_t>(hw, (n + grain - 1) / std::max<uint64_t>(grain, 1));
  if (chunks <= 1) {
    if (n) body(0, n);
    return;
  }
  std::vector<std::thread> pool;
  uint64_t step = (n + chunks - 1) / chunks;
  for (uint64_t c = 0; c < chunks; ++c) {
    uint64_t b = c * step, e = std::min(n, b + step);
    if (b >= e) break;
    pool.emplace_back([&body, b, e] { body(b, e); });
  }
  for (auto& t : pool) t.join();
}

uint64_t HostGraph::max_degree() const {
  uint64_t best = 0;
  for (uint32_t u = 0; u < n; ++u) best = std::max(best, degree(u));
  return best;
}

namespace {

// Sort u64 keys with per-thread std::sort runs and a pairwise merge tree.
void parallel_sort(std::vector<uint64_t>& keys) {
  unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  size_t n = keys.size();
  if (n < (1u << 20) || hw == 1) {
    std::sort(keys.begin(), keys.end());
    return;
  }
  size_t runs = 1;
  while (runs * 2 <= hw) runs *= 2;
  std::vector<size_t> bounds(runs + 1);
  for (size_t r = 0; r <= runs; ++r) bounds[r] = n * r / runs;
  {
    std::vector<std::thread> pool;
    for (size_t r = 0; r < runs; ++r)
      pool.emplace_back([&, r] { std::sort(keys.begin() + bounds[r], keys.begin() + bounds[r + 1]); });
    for (auto& t : pool) t.join();
  }
  std::vector<uint64_t> tmp(n);
  std::vector<uint64_t>* src = &keys;
  std::vector<uint64_t>* dst = &tmp;
  while (runs > 1) {
    std::vector<std::thread> pool;
    std::vector<size_t> nb;
    for (size_t r = 0; r < runs; r += 2) {
      nb.push_back(bounds[r]);
      size_t b0 = bounds[r], b1 = bounds[r + 1], b2 = bounds[r + 2];
      pool.emplace_back([=] {
        std::merge(src->begin() + b0, src->begin() + b1, src->begin() + b1, src->begin() + b2,
                   dst->begin() + b0);
      });
    }
    nb.push_back(n);
    for (auto& t : pool) t.join();
    bounds = nb;
    runs /= 2;
    std::swap(src, dst);
  }
  if (src != &keys) keys.swap(*src);
}

}  // namespace

HostGraph graph_from_edges(std::vector<std::pair<uint32_t, uint32_t>>& pairs,
                           uint32_t min_vertex_count) {
  // csr_graph.cpp:46-72: normalise (u<v), n from max id (self-loops count),
  // drop loops, sort + dedup, both arcs, ascending lists.
  uint64_t n64 = min_vertex_count;
  for (auto& e : pairs) n64 = std::max<uint64_t>(n64, static_cast<uint64_t>(std::max(e.first, e.second)) + 1);
  if (n64 > UINT32_MAX) throw std::invalid_argument("vertex count out of range");
  std::vector<uint64_t> keys;
  keys.reserve(pairs.size());
  for (auto& e : pairs) {
    uint32_t a = std::min(e.first, e.second), b = std::max(e.first, e.second);
    if (a != b) keys.push_back((static_cast<uint64_t>(a) << 32) | b);
  }
  std::vector<std::pair<uint32_t, uint32_t>>().swap(pairs);
  parallel_sort(keys);
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());

  HostGraph g;
  g.n = static_cast<uint32_t>(n64);
  g.edge_count = keys.size();
  g.offsets.assign(static_cast<size_t>(g.n) + 1, 0);
  for (uint64_t k : keys) {
    ++g.offsets[(k >> 32) + 1];
    ++g.offsets[(k & 0xffffffffu) + 1];
  }
  for (size_t i = 1; i < g.offsets.size(); ++i) g.offsets[i] += g.offsets[i - 1];
  g.neighbors.resize(g.offsets.back());
  std::vector<uint64_t> cur(g.offsets.begin(), g.offsets.end() - 1);
  // keys ascending by (u, v): every vertex receives its lower neighbours (as
  // the v of earlier keys) before its upper ones, each group ascending.
  for (uint64_t k : keys) {
    uint32_t u = static_cast<uint32_t>(k >> 32), v = static_cast<uint32_t>(k);
    g.neighbors[cur[u]++] = v;
    g.neighbors[cur[v]++] = u;
  }
  return g;
}

// ------------------------------------------------------------------ binary I/O
namespace {
constexpr char kMagic[4] = {'A', 'G', 'P', 'M'};

template <class T>
void put_le(std::ostream& out, T value) {
  unsigned char buf[sizeof(T)];
  for (size_t i = 0; i < sizeof(T); ++i) buf[i] = static_cast<unsigned char>(value >> (8 * i));
  out.write(reinterpret_cast<const char*>(buf), sizeof(T));
}

template <class T>
T get_le(std::istream& in) {
  unsigned char buf[sizeof(T)];
  in.read(reinterpret_cast<char*>(buf), sizeof(T));
  if (!in) throw io_error("truncated binary CSR file");
  T v = 0;
  for (size_t i = 0; i < sizeof(T); ++i) v |= static_cast<T>(buf[i]) << (8 * i);
  return v;
}

bool little_endian() {
  uint16_t x = 1;
  return *reinterpret_cast<uint8_t*>(&x) == 1;
}

HostGraph load_binary(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw io_error("cannot open graph file: " + path);
  char magic[4];
  f.read(magic, 4);
  if (!f || std::memcmp(magic, kMagic, 4) != 0) throw io_error("not a binary CSR file: " + path);
  if (get_le<uint32_t>(f) != 1) throw io_error("unsupported binary CSR version");
  uint64_t n64 = get_le<uint64_t>(f);
  uint64_t m = get_le<uint64_t>(f);
  if (n64 > UINT32_MAX) throw io_error("vertex count out of range");
  HostGraph g;
  g.n = static_cast<uint32_t>(n64);
  g.edge_count = m;
  g.offsets.resize(n64 + 1);
  if (little_endian()) {
    f.read(reinterpret_cast<char*>(g.offsets.data()), static_cast<std::streamsize>(8 * (n64 + 1)));
    if (!f) throw io_error("truncated binary CSR file");
    g.neighbors.resize(g.offsets.back());
    f.read(reinterpret_cast<char*>(g.neighbors.data()),
           static_cast<std::streamsize>(4 * g.neighbors.size()));
    if (!f) throw io_error("truncated binary CSR file");
  } else {
    for (auto& o : g.offsets) o = get_le<uint64_t>(f);
    g.neighbors.resize(g.offsets.back());
    for (auto& v : g.neighbors) v = get_le<uint32_t>(f);
  }
  return g;
}

HostGraph load_edge_list(std::istream& in) {
  // csr_graph.cpp:74-93 (same comment rules, messages and range checks)
  std::vector<std::pair<uint32_t, uint32_t>> edges;
  std::string line;
  size_t line_no = 0;
  while (std::getline(in, line)) {
    ++line_no;
    size_t start = line.find_first_not_of(" \t\r");
    if (start == std::string::npos) continue;
    if (line[start] == '#' || line[start] == '%') continue;
    std::istringstream ls(line);
    unsigned long long a, b;
    if (!(ls >> a >> b))
      throw parse_error("edge list line " + std::to_string(line_no) + ": expected two vertex ids");
    std::string extra;
    if (ls >> extra)
      throw parse_error("edge list line " + std::to_string(line_no) + ": trailing token '" + extra + "'");
    if (a > UINT32_MAX || b > UINT32_MAX)
      throw parse_error("edge list line " + std::to_string(line_no) + ": vertex id out of range");
    edges.emplace_back(static_cast<uint32_t>(a), static_cast<uint32_t>(b));
  }
  return graph_from_edges(edges, 0);
}
}  // namespace

void write_binary(const HostGraph& g, const std::string& path) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw io_error("cannot write file: " + path);
  f.write(kMagic, 4);
  put_le<uint32_t>(f, 1);
  put_le<uint64_t>(f, g.n);
  put_le<uint64_t>(f, g.edge_count);
  if (little_endian()) {
    f.write(reinterpret_cast<const char*>(g.offsets.data()),
            static_cast<std::streamsize>(8 * g.offsets.size()));
    f.write(reinterpret_cast<const char*>(g.neighbors.data()),
            static_cast<std::streamsize>(4 * g.neighbors.size()));
  } else {
    for (uint64_t o : g.offsets) put_le<uint64_t>(f, o);
    for (uint32_t v : g.neighbors) put_le<uint32_t>(f, v);
  }
  if (!f) throw io_error("write failed: " + path);
}

HostGraph load_auto(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw io_error("cannot open graph file: " + path);
  char magic[4] = {0, 0, 0, 0};
  f.read(magic, 4);
  f.close();
  if (std::memcmp(magic, kMagic, 4) == 0) return load_binary(path);
  std::ifstream t(path);
  if (!t) throw io_error("cannot open graph file: " + path);
  return load_edge_list(t);
}

// ------------------------------------------------------------------ relabel / orient
HostGraph relabel_by_degree(const HostGraph& g) {
  const uint32_t n = g.n;
  std::vector<uint32_t> order(n);
  std::iota(order.begin(), order.end(), 0u);
  // counting sort by degree keeps id order within a degree: rank of (deg, id)
  uint64_t maxd = g.max_degree();
  std::vector<uint64_t> bucket(maxd + 2, 0);
  for (uint32_t u = 0; u < n; ++u) ++bucket[g.degree(u) + 1];
  for (size_t i = 1; i < bucket.size(); ++i) bucket[i] += bucket[i - 1];
  for (uint32_t u = 0; u < n; ++u) order[bucket[g.degree(u)]++] = u;
  std::vector<uint32_t> new_id(n);
  for (uint32_t i = 0; i < n; ++i) new_id[order[i]] = i;

  HostGraph r;
  r.n = n;
  r.edge_count = g.edge_count;
  r.oriented = g.oriented;
  r.offsets.assign(static_cast<size_t>(n) + 1, 0);
  for (uint32_t i = 0; i < n; ++i) r.offsets[i + 1] = r.offsets[i] + g.degree(order[i]);
  r.neighbors.resize(r.offsets.back());
  parallel_for(n, 4096, [&](uint64_t b, uint64_t e) {
    for (uint64_t i = b; i < e; ++i) {
      uint32_t old = order[i];
      uint32_t* dst = r.neighbors.data() + r.offsets[i];
      const uint32_t* src = g.neighbors.data() + g.offsets[old];
      uint64_t d = g.degree(old);
      for (uint64_t j = 0; j < d; ++j) dst[j] = new_id[src[j]];
      std::sort(dst, dst + d);
    }
  });
  return r;
}

HostGraph orient_by_degree(const HostGraph& g) {
  const uint32_t n = g.n;
  auto less = [&](uint32_t u, uint32_t v) {
    uint64_t du = g.degree(u), dv = g.degree(v);
    return du < dv || (du == dv && u < v);
  };
  HostGraph o;
  o.n = n;
  o.edge_count = g.edge_count;
  o.oriented = true;
  o.offsets.assign(static_cast<size_t>(n) + 1, 0);
  parallel_for(n, 4096, [&](uint64_t b, uint64_t e) {
    for (uint64_t u = b; u < e; ++u) {
      uint64_t c = 0;
      for (uint64_t j = g.offsets[u]; j < g.offsets[u + 1]; ++j)
        if (less(static_cast<uint32_t>(u), g.neighbors[j])) ++c;
      o.offsets[u + 1] = c;
    }
  });
  for (size_t i = 1; i < o.offsets.size(); ++i) o.offsets[i] += o.offsets[i - 1];
  o.neighbors.resize(o.offsets.back());
  parallel_for(n, 4096, [&](uint64_t b, uint64_t e) {
    for (uint64_t u = b; u < e; ++u) {
      uint64_t at = o.offsets[u];
      for (uint64_t j = g.offsets[u]; j < g.offsets[u + 1]; ++j)
        if (less(static_cast<uint32_t>(u), g.neighbors[j])) o.neighbors[at++] = g.neighbors[j];
    }
  });
  return o;
}

// ------------------------------------------------------------------ generators
HostGraph gen_er_pairs(uint32_t n, double p, uint64_t seed) {
  // test_graphs.hpp:37-43: every pair u<v kept iff edge_keep_decision(seed,u,v,p)
  unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  std::vector<std::vector<std::pair<uint32_t, uint32_t>>> parts(hw);
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < hw; ++t)
    pool.emplace_back([&, t] {
      for (uint64_t u = t; u < n; u += hw)
        for (uint32_t v = static_cast<uint32_t>(u) + 1; v < n; ++v)
          if (edge_keep_decision(seed, static_cast<uint32_t>(u), v, p))
            parts[t].emplace_back(static_cast<uint32_t>(u), v);
    });
  for (auto& t : pool) t.join();
  std::vector<std::pair<uint32_t, uint32_t>> edges;
  for (auto& part : parts) edges.insert(edges.end(), part.begin(), part.end());
  return graph_from_edges(edges, n);
}

HostGraph gen_er_fast(uint32_t n, uint64_t target_edges, uint64_t seed, uint32_t planted_k,
                      uint32_t planted_count) {
  if (n < 2) throw std::invalid_argument("er_fast needs n >= 2");
  std::vector<std::pair<uint32_t, uint32_t>> edges(target_edges);
  parallel_for(target_edges, 1 << 16, [&](uint64_t b, uint64_t e) {
    for (uint64_t i = b; i < e; ++i) {
      CounterRng rng(seed, 0x6572ull /* "er" */, i);
      edges[i].first = static_cast<uint32_t>(rng.next_below(n));
      edges[i].second = static_cast<uint32_t>(rng.next_below(n));
    }
  });
  if (planted_k >= 2) {
    if (planted_k > n) throw std::invalid_argument("planted clique larger than the graph");
    for (uint32_t c = 0; c < planted_count; ++c) {
      CounterRng rng(seed, 0x706c616e74ull /* "plant" */, c);
      std::vector<uint32_t> vs;
      while (vs.size() < planted_k) {
        auto v = static_cast<uint32_t>(rng.next_below(n));
        if (std::find(vs.begin(), vs.end(), v) == vs.end()) vs.push_back(v);
      }
      for (uint32_t a = 0; a < planted_k; ++a)
        for (uint32_t b = a + 1; b < planted_k; ++b) edges.emplace_back(vs[a], vs[b]);
    }
  }
  return graph_from_edges(edges, n);
}

HostGraph gen_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                   uint64_t seed) {
  if (scale < 1 || scale > 31) throw std::invalid_argument("rmat scale must be in [1,31]");
  const uint64_t m = static_cast<uint64_t>(edge_factor) << scale;
  const double ab = a + b, abc = a + b + c;
  std::vector<std::pair<uint32_t, uint32_t>> edges(m);
  parallel_for(m, 1 << 16, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo; i < hi; ++i) {
      CounterRng rng(seed, 0x726d6174ull /* "rmat" */, i);
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
      edges[i] = {u, v};
    }
  });
  return graph_from_edges(edges, 1u << scale);
}

}  // namespace agpm_b200
