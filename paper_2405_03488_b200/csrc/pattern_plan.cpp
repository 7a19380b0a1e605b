// Pattern model and plan compiler (host side of the hot path, SURVEY §8(a)
// row 10). Output: agpm_plan, the field-for-field image of the reference's
// ExecutionPlan (plan.hpp:34-55); tests/test_cpu_host.py checks every builtin x
// verify mode x symmetry setting, custom specs and the error messages against
// plans dumped from the compiled reference (tests/golden/plans.json).
//
// Everything is done on adjacency bitmasks (k <= 9, one u32 row per pattern
// vertex): the edge list is the set bits of the upper triangle in row order
// (= the reference's sorted, de-duplicated edge list, pattern.cpp:24-41), the
// automorphism group comes from a pruned backtracking search over partial
// permutations instead of scanning all k! orderings (pattern.cpp:43-57 tests
// every permutation), orbits and stabilisers are masks over that group
// (Grochow-Kellis, plan.cpp:20-38), and the matching order is a greedy
// max-popcount choice over the bound mask (plan.cpp:40-76). Interface
// behaviour — plan contents, element order of every list, error texts — is
// the reference's; the implementation is not.

#include <algorithm>
#include <array>
#include <cctype>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "common.hpp"

namespace agpm_b200 {

namespace {

using Perm = std::array<int8_t, AGPM_MAX_K>;

struct Shape {
  std::string name;
  int k = 0;
  uint32_t row[AGPM_MAX_K] = {};  // row[v] bit u <=> edge {u, v}
  bool induced = false;

  bool edge(int a, int b) const { return (row[a] >> b) & 1u; }
  int deg(int v) const { return __builtin_popcount(row[v]); }
  int edge_count() const {
    int m = 0;
    for (int v = 0; v < k; ++v) m += deg(v);
    return m / 2;
  }
  // visit edges (a < b) in ascending (a, b) order
  template <class F>
  void each_edge(F&& f) const {
    for (int a = 0; a < k; ++a)
      for (uint32_t up = row[a] >> (a + 1), b = a + 1; up; up >>= 1, ++b)
        if (up & 1u) f(a, static_cast<int>(b));
  }
};

// ---------------------------------------------------------------- construction
// Raw edge pairs -> validated bitmask shape (pattern.cpp:10-41 semantics and messages)
Shape build(const std::string& name, int k, const std::vector<std::pair<int, int>>& pairs, bool induced) {
  if (k < 2 || k > AGPM_MAX_K) throw pattern_error("pattern must have between 2 and 9 vertices");
  Shape s;
  s.name = name;
  s.k = k;
  s.induced = induced;
  for (const auto& e : pairs) {
    if (e.first == e.second) throw pattern_error("pattern has a self-loop");
    if (std::min(e.first, e.second) < 0 || std::max(e.first, e.second) >= k)
      throw pattern_error("pattern edge endpoint out of range");
    s.row[e.first] |= 1u << e.second;
    s.row[e.second] |= 1u << e.first;
  }
  // connectivity: grow the component of vertex 0 until it stops changing
  uint32_t comp = 1u, prev = 0u;
  while (comp != prev) {
    prev = comp;
    for (int v = 0; v < k; ++v)
      if ((comp >> v) & 1u) comp |= s.row[v];
  }
  if (comp != (1u << k) - 1u) throw pattern_error("pattern must be connected");
  return s;
}

// std::stoi semantics for the custom-spec fields: leading blanks, optional
// sign, >= 1 digit, trailing text ignored, int range
bool parse_int(const std::string& txt, int* out) {
  const char* c = txt.c_str();
  while (*c && std::isspace(static_cast<unsigned char>(*c))) ++c;
  const bool neg = *c == '-';
  if (*c == '+' || *c == '-') ++c;
  if (!std::isdigit(static_cast<unsigned char>(*c))) return false;
  long long v = 0;
  for (; std::isdigit(static_cast<unsigned char>(*c)); ++c)
    if ((v = v * 10 + (*c - '0')) > 2147483648ll) return false;
  if (!neg && v == 2147483648ll) return false;
  *out = static_cast<int>(neg ? -v : v);
  return true;
}

// "a-b,c-d,..." -> pairs (pattern.cpp:150-160 field rules)
std::vector<std::pair<int, int>> parse_edges(const std::string& list) {
  std::vector<std::pair<int, int>> out;
  size_t at = 0;
  while (at < list.size()) {
    size_t comma = list.find(',', at);
    if (comma == std::string::npos) comma = list.size();
    const std::string item = list.substr(at, comma - at);
    at = comma + 1;
    const size_t dash = item.find('-');
    if (dash == std::string::npos) throw pattern_error("custom edge must look like a-b");
    int a = 0, b = 0;
    if (!parse_int(item.substr(0, dash), &a) || !parse_int(item.substr(dash + 1), &b))
      throw pattern_error("custom edge endpoint is not a number");
    out.emplace_back(a, b);
  }
  return out;
}

struct Builtin {
  const char* name;
  int k;
  const char* edges;  // "" = clique on k vertices
  bool induced;
};
// the reference's catalogue and its listing order (pattern.cpp:97-139)
constexpr Builtin kBuiltins[] = {
    {"triangle", 3, "", false},
    {"4clique", 4, "", false},
    {"5clique", 5, "", false},
    {"6clique", 6, "", false},
    {"7clique", 7, "", false},
    {"8clique", 8, "", false},
    {"9clique", 9, "", false},
    {"4cycle", 4, "0-1,1-2,2-3,3-0", false},
    {"5path", 5, "0-1,1-2,2-3,3-4", false},
    {"house", 5, "0-1,1-2,2-3,3-0,0-4,1-4", false},
    {"dumbbell", 6, "0-1,0-2,1-2,3-4,3-5,4-5,2-3", false},
    {"3motif-wedge", 3, "0-1,1-2", true},
    {"3motif-triangle", 3, "", true},
    {"4motif-path", 4, "0-1,1-2,2-3", true},
    {"4motif-star", 4, "0-1,0-2,0-3", true},
    {"4motif-cycle", 4, "0-1,1-2,2-3,3-0", true},
    {"4motif-tailedtriangle", 4, "0-1,0-2,1-2,1-3", true},
    {"4motif-diamond", 4, "0-1,0-2,1-2,1-3,2-3", true},
    {"4motif-clique", 4, "", true},
};

Shape from_builtin(const std::string& name) {
  for (const Builtin& b : kBuiltins) {
    if (name != b.name) continue;
    std::vector<std::pair<int, int>> pairs;
    if (*b.edges) {
      pairs = parse_edges(b.edges);
    } else {
      for (int x = 0; x < b.k; ++x)
        for (int y = x + 1; y < b.k; ++y) pairs.emplace_back(x, y);
    }
    return build(b.name, b.k, pairs, b.induced);
  }
  std::string msg = "unknown pattern '" + name + "'; valid names:";
  for (const Builtin& b : kBuiltins) msg += std::string(" ") + b.name;
  throw pattern_error(msg + " or custom:k:a-b,a-b,...");
}

Shape parse_spec(const std::string& spec, const std::string& induced) {  // pattern.cpp:130-165
  Shape s;
  static const std::string kCustom = "custom:";
  if (spec.compare(0, kCustom.size(), kCustom) == 0) {
    const std::string body = spec.substr(kCustom.size());
    const size_t colon = body.find(':');
    if (colon == std::string::npos) throw pattern_error("custom pattern needs custom:k:edges");
    int k = 0;
    if (!parse_int(body.substr(0, colon), &k)) throw pattern_error("custom pattern vertex count is not a number");
    s = build("custom", k, parse_edges(body.substr(colon + 1)), false);
  } else {
    s = from_builtin(spec);
  }
  if (induced == "edge" || induced == "vertex")
    s.induced = induced == "vertex";
  else if (!induced.empty())
    throw pattern_error("induced mode must be 'edge' or 'vertex'");
  return s;
}

// ---------------------------------------------------------------- symmetry
// All edge-preserving permutations: vertex v is mapped after 0..v-1, and a
// partial map survives only while every edge (and non-edge) among the mapped
// vertices is preserved — an automorphism is a bijection preserving adjacency
// in both directions, so this prunes to exactly the group.
void extend_auto(const Shape& s, Perm& p, uint32_t used, int v, std::vector<Perm>& out) {
  if (v == s.k) {
    out.push_back(p);
    return;
  }
  for (int img = 0; img < s.k; ++img) {
    if ((used >> img) & 1u || s.deg(img) != s.deg(v)) continue;
    bool ok = true;
    for (int u = 0; u < v && ok; ++u) ok = s.edge(u, v) == s.edge(p[u], img);
    if (!ok) continue;
    p[v] = static_cast<int8_t>(img);
    extend_auto(s, p, used | (1u << img), v + 1, out);
  }
}

std::vector<Perm> automorphism_group(const Shape& s) {
  std::vector<Perm> g;
  Perm p{};
  extend_auto(s, p, 0u, 0, g);
  return g;
}

// Grochow-Kellis symmetry breaking walked in matching order (plan.cpp:20-38):
// at each vertex u, constrain u below every other member of its orbit under
// the group fixing the earlier vertices, then restrict to u's stabiliser.
std::vector<std::pair<int, int>> orbit_constraints(const Shape& s, const std::vector<int>& order) {
  std::vector<Perm> grp = automorphism_group(s);
  std::vector<std::pair<int, int>> out;
  for (int u : order) {
    if (grp.size() < 2) break;
    uint32_t orbit = 0;
    for (const Perm& a : grp) orbit |= 1u << a[u];
    for (int w = 0; w < s.k; ++w)
      if (w != u && ((orbit >> w) & 1u)) out.emplace_back(u, w);
    grp.erase(std::remove_if(grp.begin(), grp.end(), [u](const Perm& a) { return a[u] != u; }), grp.end());
  }
  return out;
}

// ---------------------------------------------------------------- plan
// Matching order (plan.cpp:40-76): seed = the first edge (in edge order) with
// the largest endpoint-degree sum, its higher-degree endpoint first; then the
// unbound vertex with the most bound neighbours, ties to the smaller id.
std::vector<int> matching_order(const Shape& s) {
  int sa = -1, sb = -1, best = -1;
  s.each_edge([&](int a, int b) {
    if (s.deg(a) + s.deg(b) > best) {
      best = s.deg(a) + s.deg(b);
      sa = a;
      sb = b;
    }
  });
  if (s.deg(sb) > s.deg(sa)) std::swap(sa, sb);
  std::vector<int> order = {sa, sb};
  uint32_t bound = (1u << sa) | (1u << sb);
  while (static_cast<int>(order.size()) < s.k) {
    int pick = -1, most = -1;
    for (int v = 0; v < s.k; ++v) {
      if ((bound >> v) & 1u) continue;
      const int c = __builtin_popcount(s.row[v] & bound);
      if (c > most) {
        most = c;
        pick = v;
      }
    }
    bound |= 1u << pick;
    order.push_back(pick);
  }
  return order;
}

template <class Pairs>
void emit_pairs(const Pairs& src, int32_t* n, int32_t (*dst)[2]) {
  *n = 0;
  for (const auto& e : src) {
    dst[*n][0] = e.first;
    dst[*n][1] = e.second;
    ++*n;
  }
}

void compile(const Shape& s, bool eager, bool symmetric, agpm_plan* out) {  // plan.cpp:57-137
  const int k = s.k;
  std::memset(out, 0, sizeof(*out));
  std::snprintf(out->name, sizeof(out->name), "%s", s.name.c_str());
  out->k = k;
  out->induced = s.induced;
  std::vector<std::pair<int, int>> edges;
  s.each_edge([&](int a, int b) { edges.emplace_back(a, b); });
  emit_pairs(edges, &out->n_edges, out->edges);
  std::copy(s.row, s.row + k, out->adjacency);
  out->verify_mode = eager ? 0 : 1;
  out->symmetry_enabled = symmetric;

  const std::vector<int> order = matching_order(s);
  for (int i = 0; i < k; ++i) {
    out->order[i] = order[i];
    out->pos_of[order[i]] = i;
  }
  const std::vector<std::pair<int, int>> cons = symmetric ? orbit_constraints(s, order) : decltype(cons){};
  const uint32_t seed_pair = (1u << order[0]) | (1u << order[1]);
  auto on_seed = [&](const std::pair<int, int>& c) { return ((1u << c.first) | (1u << c.second)) == seed_pair; };
  out->seed_ordered = std::any_of(cons.begin(), cons.end(), on_seed) ? 1 : 0;
  emit_pairs(cons, &out->n_constraints, out->constraints);

  uint32_t verified[AGPM_MAX_K] = {};  // verified[a] bit b: edge {a, b} checked by a step or the seed
  verified[std::min(order[0], order[1])] |= 1u << std::max(order[0], order[1]);
  out->n_steps = k - 2;
  for (int pos = 2; pos < k; ++pos) {
    agpm_plan_step& st = out->steps[pos - 2];
    const int v = order[pos];
    st.pattern_vertex = v;
    st.tree_parent = -1;
    for (int q = 0; q < pos; ++q) {
      if (s.edge(v, order[q]))
        st.in_positions[st.n_in++] = q;
      else if (s.induced && eager)
        st.out_positions[st.n_out++] = q;
    }
    auto verify = [&](int a, int b) {
      const int lo = std::min(a, b), hi = std::max(a, b);
      st.verify_edges[st.n_verify][0] = lo;
      st.verify_edges[st.n_verify][1] = hi;
      ++st.n_verify;
      verified[lo] |= 1u << hi;
    };
    if (!eager) {
      st.tree_parent = st.in_positions[0];
      verify(v, order[st.tree_parent]);
      continue;
    }
    for (int i = 0; i < st.n_in; ++i) verify(v, order[st.in_positions[i]]);
    for (const auto& c : cons) {  // order bounds at the later endpoint, constraint order kept
      if (c.second == v && out->pos_of[c.first] < pos) st.greater_than[st.n_gt++] = out->pos_of[c.first];
      if (c.first == v && out->pos_of[c.second] < pos) st.less_than[st.n_lt++] = out->pos_of[c.second];
    }
  }
  if (!eager) {
    std::vector<std::pair<int, int>> closure, terminal;
    for (const auto& e : edges)
      if (!((verified[e.first] >> e.second) & 1u)) closure.push_back(e);
    for (const auto& c : cons)
      if (!on_seed(c)) terminal.push_back(c);
    emit_pairs(closure, &out->n_closure, out->closure_edges);
    emit_pairs(terminal, &out->n_terminal, out->terminal_constraints);
  }
}

void copy_out(const std::string& text, char* buf, size_t cap) {
  if (!buf || cap <= text.size()) throw std::invalid_argument("buffer too small");
  std::memcpy(buf, text.c_str(), text.size() + 1);
}

}  // namespace

// ---------------------------------------------------------------- C-ABI entry points
extern "C" {

int agpm_plan_compile(const char* spec, const char* induced, int verify_mode, int enable_symmetry,
                      agpm_plan* out) {
  return guarded([&] {
    if (!spec || !out) throw std::invalid_argument("null argument");
    if (verify_mode != 0 && verify_mode != 1) throw std::invalid_argument("verify mode must be 0 or 1");
    compile(parse_spec(spec, induced ? induced : ""), verify_mode == 0, enable_symmetry != 0, out);
  });
}

int agpm_builtin_pattern_names(char* buf, size_t cap) {
  return guarded([&] {
    std::string all;
    for (const Builtin& b : kBuiltins) all += std::string(b.name) + "\n";
    copy_out(all, buf, cap);
  });
}

int agpm_pattern_automorphism_count(const char* spec, const char* induced, uint64_t* out) {
  return guarded([&] { *out = automorphism_group(parse_spec(spec, induced ? induced : "")).size(); });
}

int agpm_plan_scaling_rule(const agpm_plan* plan, char* buf, size_t cap) {  // plan.cpp:139-148
  return guarded([&] {
    const bool eager = plan->verify_mode == 0;
    std::string rule = plan->seed_ordered ? "m" : "2m";
    for (int i = 0; i < plan->n_steps; ++i)
      rule += eager ? " * |S_" + std::to_string(i + 2) + "|" : " * c_" + std::to_string(i + 2);
    if (!eager && plan->n_closure > 0)
      rule += " (terminal closure of " + std::to_string(plan->n_closure) + " edges)";
    copy_out(rule, buf, cap);
  });
}

int agpm_plan_verifies_each_edge_once(const agpm_plan* plan, int* out) {  // plan.cpp:150-163
  // tally each checked pair in a k x k count table: the seed edge, every
  // step's verify edges, the lazy closure; the plan passes iff the checked
  // pairs are exactly the pattern's edges, each checked once
  return guarded([&] {
    int seen[AGPM_MAX_K][AGPM_MAX_K] = {};
    auto tally = [&](int a, int b) { ++seen[std::min(a, b)][std::max(a, b)]; };
    tally(plan->order[0], plan->order[1]);
    for (int i = 0; i < plan->n_steps; ++i)
      for (int e = 0; e < plan->steps[i].n_verify; ++e)
        tally(plan->steps[i].verify_edges[e][0], plan->steps[i].verify_edges[e][1]);
    for (int e = 0; e < plan->n_closure; ++e) tally(plan->closure_edges[e][0], plan->closure_edges[e][1]);
    int want[AGPM_MAX_K][AGPM_MAX_K] = {};
    for (int e = 0; e < plan->n_edges; ++e) want[plan->edges[e][0]][plan->edges[e][1]] = 1;
    bool ok = true;
    for (int a = 0; a < AGPM_MAX_K; ++a)
      for (int b = 0; b < AGPM_MAX_K; ++b) ok = ok && seen[a][b] == want[a][b];
    *out = ok;
  });
}

}  // extern "C"

}  // namespace agpm_b200
