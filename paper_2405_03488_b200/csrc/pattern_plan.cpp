// Pattern model and plan compiler (host side of the hot path, SURVEY §8(a)
// row 10). Produces agpm_plan, the field-for-field image of the reference's
// ExecutionPlan (plan.hpp:34-55). The compile rules follow plan.cpp:57-137:
//   * seed = pattern edge with the largest endpoint-degree sum, higher-degree
//     endpoint first (plan.cpp:40-53);
//   * remaining vertices by most already-bound neighbours, ties to the smaller
//     id (plan.cpp:62-76);
//   * Grochow-Kellis orbit constraints walked in matching order
//     (plan.cpp:20-38);
//   * eager steps: in-lists = bound pattern neighbours, out-lists for
//     vertex-induced patterns, order bounds at the later endpoint; lazy
//     steps: tree parent + closure + terminal constraints.
// tests/test_plan.py checks every builtin x mode x symmetry against plans
// dumped from the reference itself (tests/golden/plans.json).

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "common.hpp"

namespace agpm_b200 {

namespace {

struct Pattern {
  std::string name;
  int k = 0;
  std::vector<std::pair<int, int>> edges;
  bool vertex_induced = false;
  std::vector<uint32_t> adj;

  bool has_edge(int a, int b) const { return (adj[a] >> b) & 1u; }
  int degree(int v) const { return __builtin_popcount(adj[v]); }
  bool is_clique() const { return static_cast<int>(edges.size()) == k * (k - 1) / 2; }

  bool connected() const {  // pattern.cpp:10-22
    if (k == 0) return false;
    uint32_t reached = 1, frontier = 1;
    while (frontier) {
      uint32_t next = 0;
      for (int v = 0; v < k; ++v)
        if ((frontier >> v) & 1u) next |= adj[v];
      frontier = next & ~reached;
      reached |= next;
    }
    return reached == (1u << k) - 1;
  }

  void normalize() {  // pattern.cpp:24-41
    if (k < 2 || k > 9) throw pattern_error("pattern must have between 2 and 9 vertices");
    for (auto& [a, b] : edges) {
      if (a == b) throw pattern_error("pattern has a self-loop");
      if (a < 0 || b < 0 || a >= k || b >= k) throw pattern_error("pattern edge endpoint out of range");
      if (a > b) std::swap(a, b);
    }
    std::sort(edges.begin(), edges.end());
    edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
    adj.assign(k, 0);
    for (auto [a, b] : edges) {
      adj[a] |= 1u << b;
      adj[b] |= 1u << a;
    }
    if (!connected()) throw pattern_error("pattern must be connected");
  }

  // every permutation preserving the edge set (pattern.cpp:43-57)
  std::vector<std::vector<int>> automorphisms() const {
    std::vector<int> perm(k);
    for (int i = 0; i < k; ++i) perm[i] = i;
    std::vector<std::vector<int>> out;
    do {
      bool ok = true;
      for (auto [a, b] : edges)
        if (!has_edge(perm[a], perm[b])) {
          ok = false;
          break;
        }
      if (ok) out.push_back(perm);
    } while (std::next_permutation(perm.begin(), perm.end()));
    return out;
  }
};

Pattern make(const std::string& name, int k, std::vector<std::pair<int, int>> edges, bool vinduced) {
  Pattern p;
  p.name = name;
  p.k = k;
  p.edges = std::move(edges);
  p.vertex_induced = vinduced;
  p.normalize();
  return p;
}

std::vector<std::pair<int, int>> clique(int k) {
  std::vector<std::pair<int, int>> e;
  for (int a = 0; a < k; ++a)
    for (int b = a + 1; b < k; ++b) e.emplace_back(a, b);
  return e;
}

std::vector<std::pair<int, int>> path(int k) {
  std::vector<std::pair<int, int>> e;
  for (int a = 0; a + 1 < k; ++a) e.emplace_back(a, a + 1);
  return e;
}

const std::vector<std::string>& builtin_names() {  // pattern.cpp:97-106
  static const std::vector<std::string> names = {
      "triangle",     "4clique",        "5clique",     "6clique",     "7clique",
      "8clique",      "9clique",        "4cycle",      "5path",       "house",
      "dumbbell",     "3motif-wedge",   "3motif-triangle", "4motif-path", "4motif-star",
      "4motif-cycle", "4motif-tailedtriangle", "4motif-diamond", "4motif-clique"};
  return names;
}

Pattern builtin(const std::string& name) {  // pattern.cpp:108-139
  if (name == "triangle") return make(name, 3, clique(3), false);
  for (int k = 4; k <= 9; ++k)
    if (name == std::to_string(k) + "clique") return make(name, k, clique(k), false);
  if (name == "4cycle") return make(name, 4, {{0, 1}, {1, 2}, {2, 3}, {3, 0}}, false);
  if (name == "5path") return make(name, 5, path(5), false);
  if (name == "house") return make(name, 5, {{0, 1}, {1, 2}, {2, 3}, {3, 0}, {0, 4}, {1, 4}}, false);
  if (name == "dumbbell")
    return make(name, 6, {{0, 1}, {0, 2}, {1, 2}, {3, 4}, {3, 5}, {4, 5}, {2, 3}}, false);
  if (name == "3motif-wedge") return make(name, 3, path(3), true);
  if (name == "3motif-triangle") return make(name, 3, clique(3), true);
  if (name == "4motif-path") return make(name, 4, path(4), true);
  if (name == "4motif-star") return make(name, 4, {{0, 1}, {0, 2}, {0, 3}}, true);
  if (name == "4motif-cycle") return make(name, 4, {{0, 1}, {1, 2}, {2, 3}, {3, 0}}, true);
  if (name == "4motif-tailedtriangle") return make(name, 4, {{0, 1}, {0, 2}, {1, 2}, {1, 3}}, true);
  if (name == "4motif-diamond")
    return make(name, 4, {{0, 1}, {0, 2}, {1, 2}, {1, 3}, {2, 3}}, true);
  if (name == "4motif-clique") return make(name, 4, clique(4), true);
  std::ostringstream msg;
  msg << "unknown pattern '" << name << "'; valid names:";
  for (const auto& n : builtin_names()) msg << ' ' << n;
  msg << " or custom:k:a-b,a-b,...";
  throw pattern_error(msg.str());
}

// std::stoi semantics: optional leading whitespace and sign, at least one
// digit, trailing characters ignored; anything else throws.
bool stoi_like(const std::string& s, int* out) {
  size_t i = 0;
  while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
  bool neg = false;
  if (i < s.size() && (s[i] == '+' || s[i] == '-')) neg = s[i++] == '-';
  if (i >= s.size() || !std::isdigit(static_cast<unsigned char>(s[i]))) return false;
  long long v = 0;
  while (i < s.size() && std::isdigit(static_cast<unsigned char>(s[i]))) {
    v = v * 10 + (s[i++] - '0');
    if (v > 2147483648ll) return false;  // out_of_range
  }
  v = neg ? -v : v;
  if (v > 2147483647ll) return false;
  *out = static_cast<int>(v);
  return true;
}

Pattern parse_spec(const std::string& spec, const std::string& induced) {  // pattern.cpp:130-165
  Pattern p;
  if (spec.rfind("custom:", 0) == 0) {
    std::string rest = spec.substr(7);
    auto colon = rest.find(':');
    if (colon == std::string::npos) throw pattern_error("custom pattern needs custom:k:edges");
    int k = 0;
    if (!stoi_like(rest.substr(0, colon), &k)) throw pattern_error("custom pattern vertex count is not a number");
    std::vector<std::pair<int, int>> edges;
    std::istringstream es(rest.substr(colon + 1));
    std::string item;
    while (std::getline(es, item, ',')) {
      auto dash = item.find('-');
      if (dash == std::string::npos) throw pattern_error("custom edge must look like a-b");
      int a = 0, b = 0;
      if (!stoi_like(item.substr(0, dash), &a) || !stoi_like(item.substr(dash + 1), &b))
        throw pattern_error("custom edge endpoint is not a number");
      edges.emplace_back(a, b);
    }
    p = make("custom", k, std::move(edges), false);
  } else {
    p = builtin(spec);
  }
  if (induced == "edge")
    p.vertex_induced = false;
  else if (induced == "vertex")
    p.vertex_induced = true;
  else if (!induced.empty())
    throw pattern_error("induced mode must be 'edge' or 'vertex'");
  return p;
}

// Grochow-Kellis constraints (plan.cpp:20-38)
std::vector<std::pair<int, int>> symmetry_constraints(const Pattern& p, const std::vector<int>& order) {
  auto group = p.automorphisms();
  std::vector<std::pair<int, int>> conds;
  for (int u : order) {
    if (group.size() <= 1) break;
    std::set<int> orbit;
    for (const auto& a : group) orbit.insert(a[u]);
    if (orbit.size() > 1)
      for (int w : orbit)
        if (w != u) conds.emplace_back(u, w);
    std::vector<std::vector<int>> stab;
    for (auto& a : group)
      if (a[u] == u) stab.push_back(std::move(a));
    group = std::move(stab);
  }
  return conds;
}

std::pair<int, int> pick_seed(const Pattern& p) {  // plan.cpp:40-53
  int ba = -1, bb = -1, best = -1;
  for (auto [a, b] : p.edges) {
    int s = p.degree(a) + p.degree(b);
    if (s > best) {
      best = s;
      ba = a;
      bb = b;
    }
  }
  if (p.degree(bb) > p.degree(ba)) std::swap(ba, bb);
  return {ba, bb};
}

void put_pairs(const std::vector<std::pair<int, int>>& v, int32_t* n, int32_t (*dst)[2]) {
  *n = static_cast<int32_t>(v.size());
  for (size_t i = 0; i < v.size(); ++i) {
    dst[i][0] = v[i].first;
    dst[i][1] = v[i].second;
  }
}

void compile(const Pattern& pin, int mode, bool sym, agpm_plan* out) {  // plan.cpp:57-137
  Pattern p = pin;
  p.normalize();
  const int k = p.k;
  const bool eager = mode == 0;
  std::memset(out, 0, sizeof(*out));
  std::snprintf(out->name, sizeof(out->name), "%s", p.name.c_str());
  out->k = k;
  out->induced = p.vertex_induced;
  put_pairs(p.edges, &out->n_edges, out->edges);
  for (int v = 0; v < k; ++v) out->adjacency[v] = p.adj[v];
  out->verify_mode = eager ? 0 : 1;
  out->symmetry_enabled = sym;

  auto [s0, s1] = pick_seed(p);
  std::vector<int> order = {s0, s1};
  std::vector<bool> bound(k, false);
  bound[s0] = bound[s1] = true;
  while (static_cast<int>(order.size()) < k) {
    int best = -1, best_cnt = -1;
    for (int v = 0; v < k; ++v) {
      if (bound[v]) continue;
      int cnt = 0;
      for (int b : order)
        if (p.has_edge(v, b)) ++cnt;
      if (cnt > best_cnt) {
        best_cnt = cnt;
        best = v;
      }
    }
    bound[best] = true;
    order.push_back(best);
  }
  std::vector<int> pos_of(k, -1);
  for (int i = 0; i < k; ++i) pos_of[order[i]] = i;
  for (int i = 0; i < k; ++i) {
    out->order[i] = order[i];
    out->pos_of[i] = pos_of[i];
  }
  std::vector<std::pair<int, int>> cons;
  if (sym) cons = symmetry_constraints(p, order);
  for (auto [a, b] : cons)
    if ((a == s0 && b == s1) || (a == s1 && b == s0)) out->seed_ordered = 1;
  put_pairs(cons, &out->n_constraints, out->constraints);

  std::set<std::pair<int, int>> covered;
  covered.insert({std::min(s0, s1), std::max(s0, s1)});
  out->n_steps = k - 2;
  for (int pos = 2; pos < k; ++pos) {
    agpm_plan_step& st = out->steps[pos - 2];
    st.pattern_vertex = order[pos];
    st.tree_parent = -1;
    for (int prev = 0; prev < pos; ++prev) {
      int pv = order[prev];
      if (p.has_edge(st.pattern_vertex, pv))
        st.in_positions[st.n_in++] = prev;
      else if (p.vertex_induced && eager)
        st.out_positions[st.n_out++] = prev;
    }
    auto add_verify = [&](int a, int b) {
      st.verify_edges[st.n_verify][0] = std::min(a, b);
      st.verify_edges[st.n_verify][1] = std::max(a, b);
      ++st.n_verify;
      covered.insert({std::min(a, b), std::max(a, b)});
    };
    if (eager) {
      for (int i = 0; i < st.n_in; ++i) add_verify(st.pattern_vertex, order[st.in_positions[i]]);
      if (sym)
        for (auto [a, b] : cons) {
          if (b == st.pattern_vertex && pos_of[a] < pos) st.greater_than[st.n_gt++] = pos_of[a];
          if (a == st.pattern_vertex && pos_of[b] < pos) st.less_than[st.n_lt++] = pos_of[b];
        }
    } else {
      st.tree_parent = st.in_positions[0];
      add_verify(st.pattern_vertex, order[st.tree_parent]);
    }
  }
  if (!eager) {
    std::vector<std::pair<int, int>> closure, terminal;
    for (auto e : p.edges)
      if (!covered.count(e)) closure.push_back(e);
    for (auto [a, b] : cons) {
      bool at_seed = (a == s0 && b == s1) || (a == s1 && b == s0);
      if (!at_seed) terminal.emplace_back(a, b);
    }
    put_pairs(closure, &out->n_closure, out->closure_edges);
    put_pairs(terminal, &out->n_terminal, out->terminal_constraints);
  }
}

}  // namespace

// ---------------------------------------------------------------- C-ABI entry points
extern "C" {

int agpm_plan_compile(const char* spec, const char* induced, int verify_mode, int enable_symmetry,
                      agpm_plan* out) {
  return guarded([&] {
    if (!spec || !out) throw std::invalid_argument("null argument");
    if (verify_mode != 0 && verify_mode != 1) throw std::invalid_argument("verify mode must be 0 or 1");
    Pattern p = parse_spec(spec, induced ? induced : "");
    compile(p, verify_mode, enable_symmetry != 0, out);
  });
}

int agpm_builtin_pattern_names(char* buf, size_t cap) {
  return guarded([&] {
    std::string s;
    for (const auto& n : builtin_names()) s += n + "\n";
    if (!buf || cap <= s.size()) throw std::invalid_argument("buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

int agpm_pattern_automorphism_count(const char* spec, const char* induced, uint64_t* out) {
  return guarded([&] { *out = parse_spec(spec, induced ? induced : "").automorphisms().size(); });
}

int agpm_plan_scaling_rule(const agpm_plan* plan, char* buf, size_t cap) {  // plan.cpp:139-148
  return guarded([&] {
    std::ostringstream s;
    const bool eager = plan->verify_mode == 0;
    s << (plan->seed_ordered ? "m" : "2m");
    for (int i = 0; i < plan->n_steps; ++i) s << (eager ? " * |S_" : " * c_") << i + 2 << (eager ? "|" : "");
    if (!eager && plan->n_closure > 0) s << " (terminal closure of " << plan->n_closure << " edges)";
    std::string str = s.str();
    if (!buf || cap <= str.size()) throw std::invalid_argument("buffer too small");
    std::memcpy(buf, str.c_str(), str.size() + 1);
  });
}

int agpm_plan_verifies_each_edge_once(const agpm_plan* plan, int* out) {  // plan.cpp:150-163
  return guarded([&] {
    std::map<std::pair<int, int>, int> seen;
    int s0 = plan->order[0], s1 = plan->order[1];
    seen[{std::min(s0, s1), std::max(s0, s1)}]++;
    for (int i = 0; i < plan->n_steps; ++i)
      for (int e = 0; e < plan->steps[i].n_verify; ++e)
        seen[{plan->steps[i].verify_edges[e][0], plan->steps[i].verify_edges[e][1]}]++;
    for (int e = 0; e < plan->n_closure; ++e)
      seen[{plan->closure_edges[e][0], plan->closure_edges[e][1]}]++;
    bool ok = static_cast<int>(seen.size()) == plan->n_edges;
    for (int e = 0; ok && e < plan->n_edges; ++e) {
      auto it = seen.find({plan->edges[e][0], plan->edges[e][1]});
      ok = it != seen.end() && it->second == 1;
    }
    *out = ok;
  });
}

}  // extern "C"

}  // namespace agpm_b200
