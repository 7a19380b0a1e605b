/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the ScaleGPM sampling hot path.
 *
 * A plain-C restatement of the reference algorithm (reference =
 * /root/reference/proj, the "agpm" C++ library), function by function, each
 * citing the reference file:line it follows. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it, and only as the checker.
 * Parity pinned: tests/test_oracle.py checks it against golden vectors produced
 * by the compiled reference itself (tests/golden/, made by
 * tests/golden/make_golden.py through oracle/_ref/libagpm_ref.so).
 *
 * Plans are passed in the agpm_plan layout of include/agpm_b200.h (a field-for-
 * field image of agpm::ExecutionPlan, plan.hpp:34-55).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "agpm_b200.h"

typedef unsigned __int128 u128;

/* ------------------------------------------------------------ rng.hpp:10-70 */
static uint64_t mix64(uint64_t z) { /* rng.hpp:10-17 */
  z ^= z >> 30;
  z *= 0xbf58476d1ce4e5b9ull;
  z ^= z >> 27;
  z *= 0x94d049bb133111ebull;
  z ^= z >> 31;
  return z;
}

uint64_t orc_derive_key(uint64_t seed, uint64_t s1, uint64_t s2) { /* rng.hpp:19-24 */
  uint64_t h = mix64(seed + 0x9e3779b97f4a7c15ull);
  h = mix64(h ^ (s1 + 0xbf58476d1ce4e5b9ull));
  h = mix64(h ^ (s2 + 0x94d049bb133111ebull));
  return h;
}

typedef struct {
  uint64_t key, ctr, id;
  int philox; /* 0: the reference's CounterRng; 1: the builder's optional Philox policy */
} orc_rng;

static orc_rng rng_make(uint64_t seed, uint64_t s1, uint64_t s2) { /* rng.hpp:28-29 */
  orc_rng r = {orc_derive_key(seed, s1, s2), 0, 0, 0};
  return r;
}

/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11): ten rounds of
 * (hi, lo) = M * c for c0, c2 with M = 0xD2511F53 / 0xCD9E8D57, the outputs
 * recombined with c1, c3 and the key, the key bumped by the Weyl constants
 * 0x9E3779B9 / 0xBB67AE85 between rounds. Restated for the device's optional
 * Philox stream (csrc/rng.cuh); not part of the reference. */
void orc_philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
    c[1] = (uint32_t)p1;
    c[3] = (uint32_t)p0;
    c[0] = n0;
    c[2] = n2;
  }
}

/* the device's Philox stream: draw t of sample id under seed s is block
 * (counter (t, id), key s), low 64 bits */
static orc_rng rng_make_philox(uint64_t seed, uint64_t id) {
  orc_rng r = {seed, 0, id, 1};
  return r;
}

static uint64_t rng_u64(orc_rng* r) { /* rng.hpp:31-34 */
  if (r->philox) {
    uint32_t c[4] = {(uint32_t)r->ctr, (uint32_t)(r->ctr >> 32), (uint32_t)r->id, (uint32_t)(r->id >> 32)};
    ++r->ctr;
    orc_philox4x32_10(c, (uint32_t)r->key, (uint32_t)(r->key >> 32));
    return (uint64_t)c[0] | ((uint64_t)c[1] << 32);
  }
  r->ctr += 0x9e3779b97f4a7c15ull;
  return mix64(r->key ^ r->ctr);
}
static double rng_double(orc_rng* r) { /* rng.hpp:37 */
  return (double)(rng_u64(r) >> 11) * 0x1.0p-53;
}
static uint64_t rng_below(orc_rng* r, uint64_t n) { /* rng.hpp:40-51, Lemire */
  u128 m = (u128)rng_u64(r) * n;
  uint64_t lo = (uint64_t)m;
  if (lo < n) {
    uint64_t t = (0 - n) % n;
    while (lo < t) {
      m = (u128)rng_u64(r) * n;
      lo = (uint64_t)m;
    }
  }
  return (uint64_t)(m >> 64);
}

void orc_rng_u64(uint64_t seed, uint64_t s1, uint64_t s2, uint64_t count, uint64_t* out) {
  orc_rng r = rng_make(seed, s1, s2);
  for (uint64_t i = 0; i < count; ++i) out[i] = rng_u64(&r);
}
void orc_rng_below(uint64_t seed, uint64_t s1, uint64_t s2, uint64_t bound, uint64_t count,
                   uint64_t* out) {
  orc_rng r = rng_make(seed, s1, s2);
  for (uint64_t i = 0; i < count; ++i) out[i] = rng_below(&r, bound);
}
void orc_rng_double(uint64_t seed, uint64_t s1, uint64_t s2, uint64_t count, double* out) {
  orc_rng r = rng_make(seed, s1, s2);
  for (uint64_t i = 0; i < count; ++i) out[i] = rng_double(&r);
}
int orc_edge_keep(uint64_t seed, uint32_t u, uint32_t v, double p) { /* rng.hpp:60-65 */
  uint32_t a = u < v ? u : v, b = u < v ? v : u;
  uint64_t h = orc_derive_key(seed, a, b);
  return (double)(h >> 11) * 0x1.0p-53 < p;
}
uint32_t orc_vertex_color(uint64_t seed, uint32_t v, uint32_t c) { /* rng.hpp:67-70 */
  uint64_t h = orc_derive_key(seed, v, 0x636f6c6f72ull);
  return (uint32_t)(((u128)h * c) >> 64);
}

/* ------------------------------------------------------------ stats.cpp:8-70 */
double orc_norm_cdf(double z) { return 0.5 * erfc(-z / sqrt(2.0)); } /* stats.cpp:8 */

static double inv_norm_cdf_approx(double q) { /* stats.cpp:14-43, Acklam */
  static const double a[] = {-3.969683028665376e+01, 2.209460984245205e+02,
                             -2.759285104469687e+02, 1.383577518672690e+02,
                             -3.066479806614716e+01, 2.506628277459239e+00};
  static const double b[] = {-5.447609879822406e+01, 1.615858368580409e+02,
                             -1.556989798598866e+02, 6.680131188771972e+01,
                             -1.328068155288572e+01};
  static const double c[] = {-7.784894002430293e-03, -3.223964580411365e-01,
                             -2.400758277161838e+00, -2.549732539343734e+00,
                             4.374664141464968e+00,  2.938163982698783e+00};
  static const double d[] = {7.784695709041462e-03, 3.224671290700398e-01,
                             2.445134137142996e+00, 3.754408661907416e+00};
  const double q_low = 0.02425;
  if (q < q_low) {
    double r = sqrt(-2.0 * log(q));
    return (((((c[0] * r + c[1]) * r + c[2]) * r + c[3]) * r + c[4]) * r + c[5]) /
           ((((d[0] * r + d[1]) * r + d[2]) * r + d[3]) * r + 1.0);
  }
  if (q > 1.0 - q_low) {
    double r = sqrt(-2.0 * log(1.0 - q));
    return -(((((c[0] * r + c[1]) * r + c[2]) * r + c[3]) * r + c[4]) * r + c[5]) /
           ((((d[0] * r + d[1]) * r + d[2]) * r + d[3]) * r + 1.0);
  }
  double r = q - 0.5, t = r * r;
  return (((((a[0] * t + a[1]) * t + a[2]) * t + a[3]) * t + a[4]) * t + a[5]) * r /
         (((((b[0] * t + b[1]) * t + b[2]) * t + b[3]) * t + b[4]) * t + 1.0);
}

int orc_inv_norm_cdf(double q, double* out) { /* stats.cpp:45-55 */
  if (!(q > 0.0) || !(q < 1.0)) return AGPM_E_INVALID;
  double z = inv_norm_cdf_approx(q);
  for (int i = 0; i < 2; ++i) {
    double err = orc_norm_cdf(z) - q;
    double pdf = exp(-0.5 * z * z) / sqrt(2.0 * M_PI);
    if (pdf <= 0.0) break;
    z -= err / pdf;
  }
  *out = z;
  return AGPM_OK;
}

static void acc_add(agpm_accumulator* a, double v, int hit) { /* stats.hpp:22-27 */
  ++a->n;
  if (hit) ++a->hits;
  a->sum += v;
  a->squared_sum += v * v;
}

int orc_predicted_error(const agpm_accumulator* acc, double delta, agpm_report* rep) {
  /* stats.cpp:57-70 */
  if (!(delta > 0.0) || !(delta < 1.0)) return AGPM_E_INVALID;
  memset(rep, 0, sizeof(*rep));
  rep->epsilon_hat = INFINITY;
  rep->n = acc->n;
  if (acc->n == 0) return AGPM_OK;
  rep->hit_rate = (double)acc->hits / (double)acc->n;
  rep->mu = acc->sum / (double)acc->n;
  if (!(acc->sum > 0.0) || acc->n < 2) return AGPM_OK;
  double var = acc->squared_sum / (double)acc->n - rep->mu * rep->mu;
  if (var < 0.0) var = 0.0;
  rep->sigma = sqrt(var / (double)acc->n);
  double z;
  orc_inv_norm_cdf(1.0 - delta / 2.0, &z);
  rep->epsilon_hat = z * rep->sigma / rep->mu;
  return AGPM_OK;
}

/* ------------------------------------------------------------ graph view (csr_graph.hpp:23-41) */
typedef struct {
  uint32_t n;
  uint64_t m; /* edge_count */
  const uint64_t* begin;
  const uint64_t* end;
  const uint32_t* nbr;
  int oriented;
} view_t;

static view_t mkview(uint32_t n, uint64_t m, const uint64_t* begin, const uint64_t* end,
                     const uint32_t* nbr, int oriented) {
  view_t v = {n, m, begin, end ? end : begin + 1, nbr, oriented};
  return v;
}

typedef struct {
  uint32_t* d;
  size_t n, cap;
} vec_t;

static void vreserve(vec_t* v, size_t c) {
  if (c > v->cap) {
    v->cap = c < 16 ? 16 : c;
    v->d = (uint32_t*)realloc(v->d, v->cap * sizeof(uint32_t));
  }
}
static void vpush(vec_t* v, uint32_t x) {
  if (v->n == v->cap) vreserve(v, v->cap * 2 + 16);
  v->d[v->n++] = x;
}
static void vswap(vec_t* a, vec_t* b) {
  vec_t t = *a;
  *a = *b;
  *b = t;
}

/* ------------------------------------------------------------ set_ops.hpp:16-91 */
static int sorted_contains(const uint32_t* s, size_t len, uint32_t x) { /* :16-27 */
  size_t lo = 0, hi = len;
  while (lo < hi) {
    size_t mid = lo + (hi - lo) / 2;
    if (s[mid] < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo < len && s[lo] == x;
}

static void intersect_into(const uint32_t* a, size_t na, const uint32_t* b, size_t nb, vec_t* out) {
  /* :29-52 — galloping when |b|/|a| > 32, else merge; output is the same sorted set */
  out->n = 0;
  if (na > nb) {
    const uint32_t* t = a;
    a = b;
    b = t;
    size_t tn = na;
    na = nb;
    nb = tn;
  }
  if (na == 0) return;
  if (nb / na > 32) {
    for (size_t i = 0; i < na; ++i)
      if (sorted_contains(b, nb, a[i])) vpush(out, a[i]);
    return;
  }
  size_t i = 0, j = 0;
  while (i < na && j < nb) {
    if (a[i] < b[j])
      ++i;
    else if (b[j] < a[i])
      ++j;
    else {
      vpush(out, a[i]);
      ++i;
      ++j;
    }
  }
}

static void difference_into(const uint32_t* a, size_t na, const uint32_t* b, size_t nb, vec_t* out) {
  /* :55-71 */
  out->n = 0;
  size_t i = 0, j = 0;
  while (i < na && j < nb) {
    if (a[i] < b[j])
      vpush(out, a[i++]);
    else if (b[j] < a[i])
      ++j;
    else {
      ++i;
      ++j;
    }
  }
  for (; i < na; ++i) vpush(out, a[i]);
}

static void union_into(const uint32_t* a, size_t na, const uint32_t* b, size_t nb, vec_t* out) {
  /* :73-91 */
  out->n = 0;
  size_t i = 0, j = 0;
  while (i < na && j < nb) {
    if (a[i] < b[j])
      vpush(out, a[i++]);
    else if (b[j] < a[i])
      vpush(out, b[j++]);
    else {
      vpush(out, a[i]);
      ++i;
      ++j;
    }
  }
  for (; i < na; ++i) vpush(out, a[i]);
  for (; j < nb; ++j) vpush(out, b[j]);
}

/* ------------------------------------------------------------ walker.hpp:30-107 */
typedef struct {
  vec_t out, tmp;
} scratch_t;

static void build_step_candidates(const view_t* g, const agpm_plan* plan, int si,
                                  const uint32_t* binding, int nbound, int apply_bounds, scratch_t* s) {
  /* walker.hpp:30-83 */
  const agpm_plan_step* st = &plan->steps[si];
  s->out.n = 0;
  if (plan->verify_mode == 0) {
    /* lists sorted by size, stable like std::sort on (size) — set result is
       order-independent, so any tie order gives the same candidate set */
    const uint32_t* lp[AGPM_MAX_K] = {0};
    size_t ln[AGPM_MAX_K] = {0};
    int nl = st->n_in;
    for (int i = 0; i < nl; ++i) {
      uint32_t b = binding[st->in_positions[i]];
      lp[i] = g->nbr + g->begin[b];
      ln[i] = (size_t)(g->end[b] - g->begin[b]);
    }
    for (int i = 1; i < nl; ++i) /* insertion sort by size */
      for (int j = i; j > 0 && ln[j] < ln[j - 1]; --j) {
        const uint32_t* tp = lp[j];
        lp[j] = lp[j - 1];
        lp[j - 1] = tp;
        size_t tn = ln[j];
        ln[j] = ln[j - 1];
        ln[j - 1] = tn;
      }
    if (nl == 1) {
      vreserve(&s->out, ln[0]);
      memcpy(s->out.d, lp[0], ln[0] * sizeof(uint32_t));
      s->out.n = ln[0];
    } else {
      intersect_into(lp[0], ln[0], lp[1], ln[1], &s->out);
      for (int i = 2; i < nl && s->out.n; ++i) {
        intersect_into(s->out.d, s->out.n, lp[i], ln[i], &s->tmp);
        vswap(&s->out, &s->tmp);
      }
    }
    for (int i = 0; i < st->n_out; ++i) {
      if (!s->out.n) break;
      uint32_t b = binding[st->out_positions[i]];
      difference_into(s->out.d, s->out.n, g->nbr + g->begin[b], (size_t)(g->end[b] - g->begin[b]),
                      &s->tmp);
      vswap(&s->out, &s->tmp);
    }
  } else {
    for (int pos = 0; pos < nbound; ++pos) { /* walker.hpp:56-62 */
      uint32_t b = binding[pos];
      union_into(s->out.d, s->out.n, g->nbr + g->begin[b], (size_t)(g->end[b] - g->begin[b]), &s->tmp);
      vswap(&s->out, &s->tmp);
    }
  }
  uint32_t lo = 0, hi = 0xffffffffu; /* walker.hpp:64-69 */
  if (apply_bounds && plan->verify_mode == 0) {
    for (int i = 0; i < st->n_gt; ++i) {
      uint32_t b = binding[st->greater_than[i]] + 1;
      if (b > lo) lo = b;
    }
    for (int i = 0; i < st->n_lt; ++i) {
      uint32_t b = binding[st->less_than[i]];
      if (b < hi) hi = b;
    }
  }
  size_t kept = 0; /* walker.hpp:70-82 */
  for (size_t i = 0; i < s->out.n; ++i) {
    uint32_t c = s->out.d[i];
    if (c < lo || c >= hi) continue;
    int bound = 0;
    for (int q = 0; q < nbound; ++q)
      if (binding[q] == c) {
        bound = 1;
        break;
      }
    if (!bound) s->out.d[kept++] = c;
  }
  s->out.n = kept;
}

static int has_arc(const view_t* g, uint32_t u, uint32_t v) {
  return sorted_contains(g->nbr + g->begin[u], (size_t)(g->end[u] - g->begin[u]), v);
}

static int lazy_terminal_ok(const view_t* g, const agpm_plan* plan, const uint32_t* binding) {
  /* walker.hpp:88-107 */
  for (int i = 0; i < plan->n_closure; ++i) {
    uint32_t da = binding[plan->pos_of[plan->closure_edges[i][0]]];
    uint32_t db = binding[plan->pos_of[plan->closure_edges[i][1]]];
    if (!has_arc(g, da, db)) return 0;
  }
  for (int i = 0; i < plan->n_terminal; ++i)
    if (!(binding[plan->pos_of[plan->terminal_constraints[i][0]]] <
          binding[plan->pos_of[plan->terminal_constraints[i][1]]]))
      return 0;
  if (plan->induced) {
    for (int a = 0; a < plan->k; ++a)
      for (int b = a + 1; b < plan->k; ++b) {
        if ((plan->adjacency[a] >> b) & 1u) continue;
        if (has_arc(g, binding[plan->pos_of[a]], binding[plan->pos_of[b]])) return 0;
      }
  }
  return 1;
}

/* ------------------------------------------------------------ ns_engine.cpp:12-53 */
typedef struct {
  uint64_t* prefix; /* n+1 */
  uint64_t total;
} seed_index_t;

static seed_index_t seed_index(const view_t* g) { /* ns_engine.cpp:12-16 */
  seed_index_t s;
  s.prefix = (uint64_t*)malloc(((size_t)g->n + 1) * sizeof(uint64_t));
  s.prefix[0] = 0;
  for (uint32_t u = 0; u < g->n; ++u) s.prefix[u + 1] = s.prefix[u] + (g->end[u] - g->begin[u]);
  s.total = s.prefix[g->n];
  return s;
}

static void seed_arc(const view_t* g, const seed_index_t* s, uint64_t idx, uint32_t* u,
                     uint32_t* v) { /* ns_engine.cpp:18-23: upper_bound(prefix, idx) - 1 */
  size_t lo = 0, hi = (size_t)g->n + 1; /* first prefix > idx */
  while (lo < hi) {
    size_t mid = lo + (hi - lo) / 2;
    if (s->prefix[mid] <= idx)
      lo = mid + 1;
    else
      hi = mid;
  }
  *u = (uint32_t)(lo - 1);
  *v = g->nbr[g->begin[*u] + (idx - s->prefix[*u])];
}

static int draw_one(const view_t* g, const seed_index_t* si, const agpm_plan* plan, orc_rng* rng,
                    uint32_t* binding, double* value, scratch_t* s) {
  /* ns_engine.cpp:27-53; returns #bound positions; value = 0 on a miss */
  uint32_t u, v;
  seed_arc(g, si, rng_below(rng, si->total), &u, &v);
  if (plan->seed_ordered && u > v) {
    uint32_t t = u;
    u = v;
    v = t;
  }
  binding[0] = u;
  binding[1] = v;
  int nb = 2;
  double alpha = plan->seed_ordered ? (double)g->m : 2.0 * (double)g->m; /* plan.hpp:50-53 */
  *value = 0.0;
  for (int st = 0; st < plan->n_steps; ++st) {
    build_step_candidates(g, plan, st, binding, nb, 1, s);
    if (s->out.n == 0) return nb;
    alpha *= (double)s->out.n;
    uint32_t pick = s->out.d[rng_below(rng, s->out.n)];
    binding[nb++] = pick;
    if (plan->verify_mode == 1) {
      uint32_t parent = binding[plan->steps[st].tree_parent];
      if (!has_arc(g, parent, pick)) return nb;
    }
  }
  if (plan->verify_mode == 1 && !lazy_terminal_ok(g, plan, binding)) return nb;
  *value = alpha;
  return nb;
}

/* Per-sample records for stream (seed, worker, first+i): value, hit, bindings
 * (k per sample, 0xffffffff past a miss). Mirrors draw_sample (ns_engine.cpp:92-104). */
static int draw_records_impl(uint32_t n, uint64_t m, const uint64_t* begin, const uint64_t* end,
                             const uint32_t* nbr, const agpm_plan* plan, uint64_t seed, uint64_t worker,
                             uint64_t first, uint64_t count, double* values, uint8_t* hits,
                             uint32_t* bindings, int philox);

int orc_draw_records(uint32_t n, uint64_t m, const uint64_t* begin, const uint64_t* end,
                     const uint32_t* nbr, const agpm_plan* plan, uint64_t seed, uint64_t worker,
                     uint64_t first, uint64_t count, double* values, uint8_t* hits,
                     uint32_t* bindings) {
  return draw_records_impl(n, m, begin, end, nbr, plan, seed, worker, first, count, values, hits, bindings, 0);
}

/* the same records under the optional Philox stream (keyed by seed, counter (draw, id)) */
int orc_draw_records_philox(uint32_t n, uint64_t m, const uint64_t* begin, const uint64_t* end,
                            const uint32_t* nbr, const agpm_plan* plan, uint64_t seed, uint64_t first,
                            uint64_t count, double* values, uint8_t* hits, uint32_t* bindings) {
  return draw_records_impl(n, m, begin, end, nbr, plan, seed, 0, first, count, values, hits, bindings, 1);
}

static int draw_records_impl(uint32_t n, uint64_t m, const uint64_t* begin, const uint64_t* end,
                             const uint32_t* nbr, const agpm_plan* plan, uint64_t seed, uint64_t worker,
                             uint64_t first, uint64_t count, double* values, uint8_t* hits,
                             uint32_t* bindings, int philox) {
  view_t g = mkview(n, m, begin, end, nbr, 0);
  if (g.m == 0) return AGPM_E_INVALID;
  seed_index_t si = seed_index(&g);
  scratch_t s = {{0, 0, 0}, {0, 0, 0}};
  uint32_t b[AGPM_MAX_K];
  for (uint64_t i = 0; i < count; ++i) {
    orc_rng rng = philox ? rng_make_philox(seed, first + i) : rng_make(seed, worker, first + i);
    double val;
    int nb = draw_one(&g, &si, plan, &rng, b, &val, &s);
    values[i] = val;
    hits[i] = val != 0.0;
    if (bindings)
      for (int p = 0; p < plan->k; ++p) bindings[i * plan->k + p] = p < nb ? b[p] : 0xffffffffu;
  }
  free(si.prefix);
  free(s.out.d);
  free(s.tmp.d);
  return AGPM_OK;
}

/* run_fixed_budget with workers = 1 (ns_engine.cpp:142-153, run_window :64-88) */
int orc_fixed_budget(uint32_t n, uint64_t m, const uint64_t* begin, const uint64_t* end,
                     const uint32_t* nbr, const agpm_plan* plan, uint64_t budget, uint64_t seed,
                     agpm_accumulator* acc) {
  view_t g = mkview(n, m, begin, end, nbr, 0);
  if (budget < 1 || g.m == 0) return AGPM_E_INVALID;
  seed_index_t si = seed_index(&g);
  scratch_t s = {{0, 0, 0}, {0, 0, 0}};
  uint32_t b[AGPM_MAX_K];
  memset(acc, 0, sizeof(*acc));
  for (uint64_t i = 0; i < budget; ++i) {
    orc_rng rng = rng_make(seed, 0, i);
    double val;
    draw_one(&g, &si, plan, &rng, b, &val, &s);
    acc_add(acc, val, val != 0.0);
  }
  free(si.prefix);
  free(s.out.d);
  free(s.tmp.d);
  return AGPM_OK;
}

/* run_ns_online with workers = 1 (ns_engine.cpp:106-140) */
int orc_ns_online(uint32_t n, uint64_t m, const uint64_t* begin, const uint64_t* end,
                  const uint32_t* nbr, const agpm_plan* plan, double eps, double delta,
                  const agpm_online_policy* pol, uint64_t seed, agpm_online_result* out) {
  if (!(eps > 0.0) || !(eps < 1.0) || !(delta > 0.0) || !(delta < 1.0)) return AGPM_E_INVALID;
  view_t g = mkview(n, m, begin, end, nbr, 0);
  if (g.m == 0) return AGPM_E_INVALID;
  seed_index_t si = seed_index(&g);
  scratch_t s = {{0, 0, 0}, {0, 0, 0}};
  uint32_t b[AGPM_MAX_K];
  uint64_t window = pol->n_min > 10 ? pol->n_min : 10; /* max(n_min, 10*workers) */
  if (pol->profiled_n_samples > 0 && pol->profiled_n_samples / 10 > window)
    window = pol->profiled_n_samples / 10;
  memset(out, 0, sizeof(*out));
  agpm_accumulator acc = {0, 0, 0.0, 0.0};
  uint64_t drawn = 0, idx = 0;
  for (;;) {
    uint64_t this_window = pol->max_samples - drawn < window ? pol->max_samples - drawn : window;
    if (this_window == 0) break;
    for (uint64_t i = 0; i < this_window; ++i) {
      orc_rng rng = rng_make(seed, 0, idx++);
      double val;
      draw_one(&g, &si, plan, &rng, b, &val, &s);
      acc_add(&acc, val, val != 0.0);
    }
    drawn += this_window;
    ++out->windows;
    orc_predicted_error(&acc, delta, &out->report);
    out->accumulator = acc;
    if (out->report.epsilon_hat <= eps) {
      out->report.converged = 1;
      break;
    }
    if (drawn >= pol->max_samples) break;
  }
  free(si.prefix);
  free(s.out.d);
  free(s.tmp.d);
  return AGPM_OK;
}

/* Multi-threaded checker variants for the big configs (RMAT-22 … RMAT-26 parity
 * tests): each sample is still drawn by draw_one from its own stream
 * CounterRng(seed, 0, i), so per-sample records are those of the sequential
 * functions above; the online run draws a speculative block of windows in
 * parallel into a value buffer, then accumulates it SEQUENTIALLY in sample-id
 * order with the stop test after every window — bit-identical to
 * orc_ns_online (ns_engine.cpp:106-140 with workers = 1), only faster. */
int orc_draw_records_mt(uint32_t n, uint64_t m, const uint64_t* begin, const uint64_t* end,
                        const uint32_t* nbr, const agpm_plan* plan, uint64_t seed, uint64_t first,
                        uint64_t count, double* values, uint8_t* hits, uint32_t* bindings, int threads) {
  view_t g = mkview(n, m, begin, end, nbr, 0);
  if (g.m == 0) return AGPM_E_INVALID;
  seed_index_t si = seed_index(&g);
  const int64_t chunk = 256;
  const int64_t nchunks = (int64_t)((count + chunk - 1) / chunk);
#pragma omp parallel num_threads(threads > 0 ? threads : 1)
  {
    scratch_t s = {{0, 0, 0}, {0, 0, 0}};
    uint32_t b[AGPM_MAX_K];
#pragma omp for schedule(dynamic, 1)
    for (int64_t c = 0; c < nchunks; ++c) {
      uint64_t lo = (uint64_t)c * chunk, hi = lo + chunk < count ? lo + chunk : count;
      for (uint64_t i = lo; i < hi; ++i) {
        orc_rng rng = rng_make(seed, 0, first + i);
        double val;
        int nb = draw_one(&g, &si, plan, &rng, b, &val, &s);
        values[i] = val;
        hits[i] = val != 0.0;
        if (bindings)
          for (int p = 0; p < plan->k; ++p) bindings[i * plan->k + p] = p < nb ? b[p] : 0xffffffffu;
      }
    }
    free(s.out.d);
    free(s.tmp.d);
  }
  free(si.prefix);
  return AGPM_OK;
}

int orc_ns_online_mt(uint32_t n, uint64_t m, const uint64_t* begin, const uint64_t* end,
                     const uint32_t* nbr, const agpm_plan* plan, double eps, double delta,
                     const agpm_online_policy* pol, uint64_t seed, agpm_online_result* out, int threads) {
  if (!(eps > 0.0) || !(eps < 1.0) || !(delta > 0.0) || !(delta < 1.0)) return AGPM_E_INVALID;
  view_t g = mkview(n, m, begin, end, nbr, 0);
  if (g.m == 0) return AGPM_E_INVALID;
  uint64_t window = pol->n_min > 10 ? pol->n_min : 10;
  if (pol->profiled_n_samples > 0 && pol->profiled_n_samples / 10 > window)
    window = pol->profiled_n_samples / 10;
  const uint64_t block = 1ull << 17; /* samples drawn speculatively per round */
  double* vals = (double*)malloc(block * sizeof(double));
  uint8_t* hit = (uint8_t*)malloc(block);
  memset(out, 0, sizeof(*out));
  agpm_accumulator acc = {0, 0, 0.0, 0.0};
  uint64_t drawn = 0, idx = 0, have = 0, used = 0; /* buffer holds ids [idx-have, idx) */
  int done = 0;
  while (!done) {
    uint64_t this_window = pol->max_samples - drawn < window ? pol->max_samples - drawn : window;
    if (this_window == 0) break;
    for (uint64_t i = 0; i < this_window; ++i) {
      if (used == have) {
        orc_draw_records_mt(n, m, begin, end, nbr, plan, seed, idx, block, vals, hit, NULL, threads);
        idx += block;
        have = block;
        used = 0;
      }
      acc_add(&acc, vals[used], hit[used]);
      ++used;
    }
    drawn += this_window;
    ++out->windows;
    orc_predicted_error(&acc, delta, &out->report);
    out->accumulator = acc;
    if (out->report.epsilon_hat <= eps) {
      out->report.converged = 1;
      done = 1;
    } else if (drawn >= pol->max_samples) {
      done = 1;
    }
  }
  free(vals);
  free(hit);
  return AGPM_OK;
}

/* ------------------------------------------------------------ exact_engine.cpp:19-91 */
/* exact_engine.cpp:19-62 search_from_seed: the iterative DFS restated recursively */
static uint64_t dfs(const view_t* g, const agpm_plan* plan, int apply_bounds, uint32_t* binding,
                    int si, scratch_t* frames) {
  const int depth = plan->n_steps;
  scratch_t* s = &frames[si];
  build_step_candidates(g, plan, si, binding, si + 2, apply_bounds, s);
  const int last = si + 1 == depth;
  if (last && plan->verify_mode == 0) return s->out.n; /* eager leaf adds |S| (:34-37) */
  uint64_t count = 0;
  for (size_t i = 0; i < s->out.n; ++i) {
    uint32_t v = s->out.d[i];
    binding[si + 2] = v;
    if (plan->verify_mode == 1) {
      uint32_t parent = binding[plan->steps[si].tree_parent];
      if (!has_arc(g, parent, v)) continue;
    }
    if (last) {
      if (lazy_terminal_ok(g, plan, binding)) ++count;
      continue;
    }
    count += dfs(g, plan, apply_bounds, binding, si + 1, frames);
  }
  return count;
}

/* exact_engine.cpp:66-91, restricted to the seeds of one shard: arc index idx
 * (u ascending, list order — the device's seed-arc order) belongs to shard
 * (idx / 32) % nshards. nshards = 1 is the reference's exact_count. */
int orc_exact_count_shard(uint32_t n, uint64_t m, const uint64_t* begin, const uint64_t* end,
                          const uint32_t* nbr, int oriented, const agpm_plan* plan, uint32_t shard,
                          uint32_t nshards, uint64_t* count) {
  view_t g = mkview(n, m, begin, end, nbr, oriented);
  int is_clique = plan->n_edges == plan->k * (plan->k - 1) / 2;
  int oriented_clique = oriented && is_clique;
  if (oriented && !is_clique) return AGPM_E_INVALID;
  if (oriented && plan->verify_mode == 1) return AGPM_E_INVALID;
  int apply_bounds = !oriented_clique;
  scratch_t frames[AGPM_MAX_K];
  memset(frames, 0, sizeof(frames));
  uint32_t binding[AGPM_MAX_K];
  if (nshards == 0 || shard >= nshards) return AGPM_E_INVALID;
  uint64_t total = 0, idx = 0;
  for (uint32_t u = 0; u < n; ++u) {
    for (uint64_t e = g.begin[u]; e < g.end[u]; ++e, ++idx) {
      uint32_t v = g.nbr[e];
      if ((idx / 32) % nshards != shard) continue;
      if (!oriented_clique && plan->seed_ordered && u > v) continue;
      binding[0] = u;
      binding[1] = v;
      if (plan->n_steps == 0) {
        if (plan->verify_mode == 1 && !lazy_terminal_ok(&g, plan, binding)) continue;
        ++total;
        continue;
      }
      total += dfs(&g, plan, apply_bounds, binding, 0, frames);
    }
  }
  for (int i = 0; i < AGPM_MAX_K; ++i) {
    free(frames[i].out.d);
    free(frames[i].tmp.d);
  }
  *count = total;
  return AGPM_OK;
}

int orc_exact_count(uint32_t n, uint64_t m, const uint64_t* begin, const uint64_t* end,
                    const uint32_t* nbr, int oriented, const agpm_plan* plan, uint64_t* count) {
  return orc_exact_count_shard(n, m, begin, end, nbr, oriented, plan, 0, 1, count);
}

/* ------------------------------------------------------------ csr_graph.cpp:172-239 */
/* orient_by_degree (csr_graph.cpp:172-188): out arrays sized n+1 and m */
void orc_orient_by_degree(uint32_t n, const uint64_t* off, const uint32_t* nbr, uint64_t* o_off,
                          uint32_t* o_nbr) {
  o_off[0] = 0;
  for (uint32_t u = 0; u < n; ++u) {
    uint64_t du = off[u + 1] - off[u], c = 0;
    for (uint64_t e = off[u]; e < off[u + 1]; ++e) {
      uint32_t v = nbr[e];
      uint64_t dv = off[v + 1] - off[v];
      if (du < dv || (du == dv && u < v)) o_nbr[o_off[u] + c++] = v;
    }
    o_off[u + 1] = o_off[u] + c;
  }
}

/* bernoulli_sparsify (csr_graph.cpp:190-213): out arrays sized n+1 and arcs; returns kept arcs */
uint64_t orc_bernoulli_sparsify(uint32_t n, const uint64_t* off, const uint32_t* nbr, double p,
                                uint64_t seed, uint64_t* o_off, uint32_t* o_nbr) {
  o_off[0] = 0;
  for (uint32_t u = 0; u < n; ++u) {
    uint64_t c = 0;
    for (uint64_t e = off[u]; e < off[u + 1]; ++e)
      if (orc_edge_keep(seed, u, nbr[e], p)) o_nbr[o_off[u] + c++] = nbr[e];
    o_off[u + 1] = o_off[u] + c;
  }
  return o_off[n];
}

/* triangle_count (csr_graph.cpp:225-239) */
uint64_t orc_triangle_count(uint32_t n, const uint64_t* off, const uint32_t* nbr) {
  uint64_t* o_off = (uint64_t*)malloc(((size_t)n + 1) * sizeof(uint64_t));
  uint32_t* o_nbr = (uint32_t*)malloc((size_t)(off[n] / 2 + 1) * sizeof(uint32_t));
  orc_orient_by_degree(n, off, nbr, o_off, o_nbr);
  vec_t out = {0, 0, 0};
  uint64_t total = 0;
  for (uint32_t u = 0; u < n; ++u)
    for (uint64_t e = o_off[u]; e < o_off[u + 1]; ++e) {
      uint32_t v = o_nbr[e];
      intersect_into(o_nbr + o_off[u], (size_t)(o_off[u + 1] - o_off[u]), o_nbr + o_off[v],
                     (size_t)(o_off[v + 1] - o_off[v]), &out);
      total += out.n;
    }
  free(out.d);
  free(o_off);
  free(o_nbr);
  return total;
}

/* ------------------------------------------------------------ colored_csr.cpp:14-54 */
/* color_vertices + build_splits: stable partition of each list into
 * (same colour | rest). out_nbr is the permuted neighbour copy. Returns
 * same-colour edge count (same arcs / 2). */
uint64_t orc_color_split(uint32_t n, const uint64_t* off, const uint32_t* nbr, uint32_t c,
                         uint64_t seed, uint32_t* colors, uint64_t* split_end, uint32_t* out_nbr) {
  for (uint32_t v = 0; v < n; ++v) colors[v] = orc_vertex_color(seed, v, c); /* :48-54 */
  uint64_t same = 0;
  for (uint32_t u = 0; u < n; ++u) { /* :14-28 stable_partition */
    uint64_t w = off[u];
    for (uint64_t e = off[u]; e < off[u + 1]; ++e)
      if (colors[nbr[e]] == colors[u]) out_nbr[w++] = nbr[e];
    split_end[u] = w;
    same += w - off[u];
    for (uint64_t e = off[u]; e < off[u + 1]; ++e)
      if (colors[nbr[e]] != colors[u]) out_nbr[w++] = nbr[e];
  }
  return same / 2;
}

/* ------------------------------------------------------------ benchmark graph inputs */
/* The reference arm of bench.py builds its input without the product library:
 * edges from this generator, CSR by the reference's own CsrGraph::from_edges,
 * the (degree, id) relabel below, the AGPM v1 file below, then the reference's
 * load_graph_auto. tests/test_cpu_oracle.py pins the result to the product's
 * rmat(...).relabel_by_degree() array for array. */

/* The benchmark RMAT generator (the product's definition, csrc/host_graph.cpp
 * gen_rmat): edge i draws `scale` doubles from
 * CounterRng(seed, "rmat", i) (rng.hpp:28-37) and descends the quadrants
 * (a | b: v bit | c: u bit | d: both), bits appended MSB first. pairs = 2*ef<<scale u32. */
void orc_gen_rmat_pairs(uint32_t scale, uint32_t edge_factor, double a, double b, double c, uint64_t seed,
                        uint32_t* pairs) {
  const int64_t m = (int64_t)edge_factor << scale;
  const double ab = a + b, abc = a + b + c;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    orc_rng r = rng_make(seed, 0x726d6174ull /* "rmat" */, (uint64_t)i);
    uint32_t u = 0, v = 0;
    for (uint32_t l = 0; l < scale; ++l) {
      double x = rng_double(&r);
      uint32_t bu = x >= ab, bv = (x >= a && x < ab) || x >= abc;
      u = (u << 1) | bu;
      v = (v << 1) | bv;
    }
    pairs[2 * i] = u;
    pairs[2 * i + 1] = v;
  }
}

static int cmp_u32(const void* x, const void* y) {
  uint32_t a = *(const uint32_t*)x, b = *(const uint32_t*)y;
  return (a > b) - (a < b);
}

/* Relabel by (degree, id) rank (not in the reference —
 * the product's definition, csrc/host_graph.cpp relabel_by_degree): a stable
 * counting sort by degree gives order[]; vertex order[i] becomes i; each new
 * list is the old list mapped and sorted ascending. out_off n+1, out_nbr arcs. */
void orc_relabel_by_degree(uint32_t n, const uint64_t* off, const uint32_t* nbr, uint64_t* out_off,
                           uint32_t* out_nbr) {
  uint64_t maxd = 0;
  for (uint32_t u = 0; u < n; ++u)
    if (off[u + 1] - off[u] > maxd) maxd = off[u + 1] - off[u];
  uint64_t* bucket = (uint64_t*)calloc(maxd + 2, sizeof(uint64_t));
  uint32_t* order = (uint32_t*)malloc((size_t)n * sizeof(uint32_t) + 4);
  uint32_t* new_id = (uint32_t*)malloc((size_t)n * sizeof(uint32_t) + 4);
  for (uint32_t u = 0; u < n; ++u) ++bucket[off[u + 1] - off[u] + 1];
  for (uint64_t d = 1; d <= maxd + 1; ++d) bucket[d] += bucket[d - 1];
  for (uint32_t u = 0; u < n; ++u) order[bucket[off[u + 1] - off[u]]++] = u;
  for (uint32_t i = 0; i < n; ++i) new_id[order[i]] = i;
  out_off[0] = 0;
  for (uint32_t i = 0; i < n; ++i) out_off[i + 1] = out_off[i] + (off[order[i] + 1] - off[order[i]]);
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t i = 0; i < (int64_t)n; ++i) {
    const uint32_t old = order[i];
    uint32_t* dst = out_nbr + out_off[i];
    const uint64_t d = off[old + 1] - off[old];
    for (uint64_t j = 0; j < d; ++j) dst[j] = new_id[nbr[off[old] + j]];
    qsort(dst, d, sizeof(uint32_t), cmp_u32);
  }
  free(bucket);
  free(order);
  free(new_id);
}

/* write_binary_csr (csr_graph.cpp, the AGPM v1 layout): "AGPM", u32 version 1,
 * u64 n, u64 m, u64 offsets[n+1], u32 neighbors[offsets[n]], little endian
 * (this host is little endian, so the arrays are written as they lie). */
#include <stdio.h>
int orc_write_binary_csr(const char* path, uint32_t n, uint64_t m, const uint64_t* off, const uint32_t* nbr) {
  FILE* f = fopen(path, "wb");
  if (!f) return AGPM_E_IO;
  const uint32_t version = 1;
  const uint64_t n64 = n;
  int ok = fwrite("AGPM", 1, 4, f) == 4 && fwrite(&version, 4, 1, f) == 1 && fwrite(&n64, 8, 1, f) == 1 &&
           fwrite(&m, 8, 1, f) == 1 && fwrite(off, 8, (size_t)n + 1, f) == (size_t)n + 1 &&
           fwrite(nbr, 4, off[n], f) == off[n];
  ok = (fclose(f) == 0) && ok;
  return ok ? AGPM_OK : AGPM_E_IO;
}
