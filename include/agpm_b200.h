/*
 * agpm_b200.h — C-ABI boundary of the B200-native ScaleGPM sampling hot path.
 *
 * Everything here is plain C: fixed-size structs, raw pointers, sizes and an
 * int status (AGPM_OK or an AGPM_E* code) with a thread-local message from
 * agpm_last_error(). No torch or C++ types cross this line. The C++ drop-in
 * API (include/agpm/ headers, namespace agpm) and the Python mirror
 * (paper_2405_03488_b200/__init__.py) are thin wrappers over these calls.
 *
 * Each entry point names the reference interface it replaces
 * (reference = /root/reference/proj, "agpm" C++20 library).
 *
 * Stream semantics: every call that takes `void* stream` accepts a
 * cudaStream_t (NULL = the library's own non-blocking stream for the calling
 * host thread and current device; pass
 * cudaStreamLegacy, (void*)1, for the legacy default stream). Calls that return
 * host results synchronise that stream before returning; *_dev calls only
 * enqueue work.
 */
#ifndef AGPM_B200_H_
#define AGPM_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AGPM_B200_ABI_VERSION 1

/* status codes; the C++ wrapper rethrows them as the reference's exception types */
#define AGPM_OK 0
#define AGPM_E_INVALID 1   /* std::invalid_argument   (e.g. ns_engine.cpp:94-95,108-110) */
#define AGPM_E_PATTERN 2   /* agpm::pattern_error      (pattern.hpp:49-51) */
#define AGPM_E_IO 3        /* agpm::io_error           (csr_graph.hpp:15-17) */
#define AGPM_E_PARSE 4     /* agpm::parse_error        (csr_graph.hpp:12-14) */
#define AGPM_E_CUDA 5      /* device failure (no reference analogue) */
#define AGPM_E_NODEVICE 6  /* no CUDA device: the product has no CPU fallback */
#define AGPM_E_INTERNAL 7

#define AGPM_MAX_K 9
#define AGPM_MAX_PAIRS 36 /* C(9,2) */

/* ---------------------------------------------------------------- plans ---
 * Mirrors agpm::PlanStep / agpm::ExecutionPlan (plan.hpp:21-55). Position
 * lists keep the reference's element order. */
typedef struct agpm_plan_step {
  int32_t pattern_vertex;
  int32_t n_in, in_positions[AGPM_MAX_K];
  int32_t n_out, out_positions[AGPM_MAX_K];
  int32_t n_gt, greater_than[AGPM_MAX_K];
  int32_t n_lt, less_than[AGPM_MAX_K];
  int32_t tree_parent;
  int32_t n_verify, verify_edges[AGPM_MAX_K][2];
} agpm_plan_step;

typedef struct agpm_plan {
  char name[64];
  int32_t k;                /* pattern.vertex_count */
  int32_t induced;          /* 0 = Edge, 1 = Vertex (pattern.hpp:11) */
  int32_t n_edges, edges[AGPM_MAX_PAIRS][2];
  uint32_t adjacency[AGPM_MAX_K];
  int32_t verify_mode;      /* 0 = Eager, 1 = Lazy (plan.hpp:14) */
  int32_t order[AGPM_MAX_K], pos_of[AGPM_MAX_K];
  int32_t seed_ordered, symmetry_enabled;
  int32_t n_steps;
  agpm_plan_step steps[AGPM_MAX_K - 2];
  int32_t n_closure, closure_edges[AGPM_MAX_PAIRS][2];
  int32_t n_constraints, constraints[AGPM_MAX_PAIRS][2];
  int32_t n_terminal, terminal_constraints[AGPM_MAX_PAIRS][2];
} agpm_plan;

/* replaces parse_pattern_spec + compile_plan (pattern.cpp:130-165, plan.cpp:57-137).
 * induced_override: NULL/"" keep default, "edge", "vertex". */
int agpm_plan_compile(const char* spec, const char* induced_override, int verify_mode,
                      int enable_symmetry, agpm_plan* out);
/* replaces builtin_pattern_names (pattern.cpp:140-148); '\n'-separated */
int agpm_builtin_pattern_names(char* buf, size_t cap);
/* replaces Pattern::automorphisms().size() (pattern.cpp:43-57) */
int agpm_pattern_automorphism_count(const char* spec, const char* induced_override,
                                    uint64_t* out);
/* replaces ExecutionPlan::scaling_rule_text (plan.cpp:139-148) */
int agpm_plan_scaling_rule(const agpm_plan* plan, char* buf, size_t cap);
/* replaces plan_verifies_each_edge_once (plan.cpp:150-163) */
int agpm_plan_verifies_each_edge_once(const agpm_plan* plan, int* out);

/* ---------------------------------------------------------------- stats ---
 * Mirrors SampleAccumulator / ConvergenceReport (stats.hpp:16-43). */
typedef struct agpm_accumulator {
  uint64_t n, hits;
  double sum, squared_sum;
} agpm_accumulator;

typedef struct agpm_report {
  double mu, sigma, epsilon_hat;
  uint64_t n;
  int32_t converged;
  double hit_rate;
} agpm_report;

double agpm_norm_cdf(double z);                                   /* stats.cpp:8 */
int agpm_inv_norm_cdf(double q, double* out);                      /* stats.cpp:45-55 */
int agpm_predicted_error(const agpm_accumulator* acc, double delta,
                         agpm_report* out);                        /* stats.cpp:57-70 */

/* ------------------------------------------------------ host CSR graphs ---
 * Owning host CSR, mirrors agpm::CsrGraph (csr_graph.hpp:46-80): u64 offsets,
 * u32 sorted neighbours, symmetric unless oriented. */
typedef struct agpm_host_graph agpm_host_graph;

/* CsrGraph::from_edges (csr_graph.cpp:46-72); edges = 2*n_edges u32 */
int agpm_host_graph_from_edges(const uint32_t* edges, uint64_t n_edges, uint32_t min_vertex_count,
                               agpm_host_graph** out);
/* adopt/copy an existing CSR (CsrGraph ctor, csr_graph.cpp:32-38) */
int agpm_host_graph_from_csr(uint32_t n, uint64_t edge_count, const uint64_t* offsets,
                             const uint32_t* neighbors, int oriented, agpm_host_graph** out);
int agpm_host_graph_load(const char* path, agpm_host_graph** out);        /* load_graph_auto :162-170 */
int agpm_host_graph_write_binary(const agpm_host_graph* g, const char* path); /* :109-122 */
int agpm_host_graph_info(const agpm_host_graph* g, uint32_t* n, uint64_t* edge_count,
                         uint64_t* arcs, int* oriented, uint64_t* max_degree);
int agpm_host_graph_arrays(const agpm_host_graph* g, const uint64_t** offsets,
                           const uint32_t** neighbors);
void agpm_host_graph_free(agpm_host_graph* g);
/* process-unique, never-reused id of a host graph (keys device-mirror caches) */
int agpm_host_graph_generation(const agpm_host_graph* g, uint64_t* out);

/* Relabel so vertex id = rank of (degree, id): the reference's id-order
 * symmetry constraints then coincide with degree orientation. */
int agpm_host_graph_relabel_by_degree(const agpm_host_graph* g, agpm_host_graph** out);
/* orient_by_degree (csr_graph.cpp:172-188) */
int agpm_host_graph_orient_by_degree(const agpm_host_graph* g, agpm_host_graph** out);

/* Deterministic generators (all built on CounterRng, rng.hpp:26-56).
 * er_pairs: the reference test generator er_graph (test_graphs.hpp:37-43), O(n^2).
 * er_fast: G(n, m_target) by uniform pair draws, O(m).
 * rmat: scale/edge_factor/(a,b,c) quadrant recursion, undirected, dedup, no loops.
 * planted: adds `count` k-cliques on uniformly drawn vertex k-sets. */
int agpm_gen_er_pairs(uint32_t n, double p, uint64_t seed, agpm_host_graph** out);
int agpm_gen_er_fast(uint32_t n, uint64_t target_edges, uint64_t seed, uint32_t planted_k,
                     uint32_t planted_count, agpm_host_graph** out);
int agpm_gen_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                  uint64_t seed, agpm_host_graph** out);

/* ------------------------------------------------------ device graphs -----
 * Device-resident mirror of a CsrView (csr_graph.hpp:23-41). Created from
 * HOST arrays (copied over), or produced on device by sparsification. */
typedef struct agpm_graph agpm_graph;

/* end == NULL means a plain view (end[u] = begin[u+1]) */
int agpm_graph_upload(uint32_t n, uint64_t edge_count, const uint64_t* begin, const uint64_t* end,
                      const uint32_t* neighbors, uint64_t neighbor_len, int oriented, void* stream,
                      agpm_graph** out);
int agpm_graph_upload_host(const agpm_host_graph* g, void* stream, agpm_graph** out);
/* Build the view's sampling indexes now — the dense-core bit matrix (current
 * core dimension) and the twin-arc index (4 B per arc, best effort: skipped when
 * HBM is short) — instead of lazily: the core on the view's first flat / frontier
 * launch, the twin index once as many ids as the view has arcs have been sampled on it.
 * Samples are identical either way; returns when the indexes are built. */
int agpm_graph_prepare(agpm_graph* g, void* stream);
/* page-lock (cudaHostRegister) a host graph's arrays so uploads run at DMA
 * speed; unpinned automatically by agpm_host_graph_free */
int agpm_host_graph_pin(agpm_host_graph* g);
int agpm_graph_free(agpm_graph* g);
int agpm_graph_info(const agpm_graph* g, uint32_t* n, uint64_t* edge_count, uint64_t* arcs,
                    int* oriented, uint64_t* device_bytes);
/* CsrView::max_degree (csr_graph.cpp:21-25) of the device view */
int agpm_graph_max_degree(const agpm_graph* g, uint64_t* out);
/* length of the view's neighbour array (>= its arc count for split views) */
int agpm_graph_neighbor_len(const agpm_graph* g, uint64_t* len);
/* copy the view back to host (tests): begin[n], end[n], neighbors[neighbor_len] */
int agpm_graph_download(const agpm_graph* g, uint64_t* begin, uint64_t* end, uint32_t* neighbors);

/* --------------------------------------------- device graph ingest -----
 * The host builders above, run in HBM (radix sort / unique / relabel / CSR on
 * the GPU); results are bit-identical to building on the host and uploading.
 * relabel != 0 applies relabel_by_degree (rank of (degree, id)) on the way.
 *   agpm_graph_from_edges_device  CsrGraph::from_edges (csr_graph.cpp:46-72);
 *                                 pairs = host u32[2*count] (u0,v0,u1,v1,...)
 *   agpm_gen_rmat_device          == agpm_gen_rmat (+relabel) on the device
 *   agpm_gen_er_fast_device       == agpm_gen_er_fast (+relabel)
 *   agpm_graph_relabel_device     == agpm_host_graph_relabel_by_degree
 *   agpm_graph_orient_device      orient_by_degree (csr_graph.cpp:172) */
int agpm_graph_from_edges_device(const uint32_t* pairs, uint64_t count, uint32_t min_vertex_count,
                                 int relabel, void* stream, agpm_graph** out);
int agpm_gen_rmat_device(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                         uint64_t seed, int relabel, void* stream, agpm_graph** out);
int agpm_gen_er_fast_device(uint32_t n, uint64_t target_edges, uint64_t seed, uint32_t planted_k,
                            uint32_t planted_count, int relabel, void* stream, agpm_graph** out);
int agpm_graph_relabel_device(const agpm_graph* g, void* stream, agpm_graph** out);
int agpm_graph_orient_device(const agpm_graph* g, void* stream, agpm_graph** out);

/* ------------------------------------------------- neighbour sampling -----
 * Global sample id i uses CounterRng(seed, 0, i) (rng.hpp:26-56), i.e. the
 * reference's workers=1 streams (ns_engine.cpp:72): GPU results are
 * sample-identical to the reference's single-worker run for every device and
 * rank count. */
typedef struct agpm_online_policy {
  uint64_t n_min;              /* OnlinePolicy::n_min (ns_engine.hpp:40) */
  uint64_t max_samples;        /* OnlinePolicy::max_samples */
  uint64_t profiled_n_samples; /* OnlinePolicy::profiled_n_samples */
} agpm_online_policy;

typedef struct agpm_online_result {
  agpm_report report;
  agpm_accumulator accumulator;
  uint64_t windows;
  uint64_t work_units;   /* device: sample steps evaluated (not the CPU comparison count) */
  uint64_t samples_launched; /* includes speculative samples past the stop window */
  double seconds;        /* device wall time of the sampling loop */
} agpm_online_result;

/* draw_sample for ids [first_id, first_id+count) (ns_engine.cpp:92-104):
 * values[i] = scaled value (0 on a miss), hits[i] in {0,1}, bindings
 * (nullable) = count*k u32 matching-order bindings (0xffffffff past a miss). */
int agpm_ns_draw(agpm_graph* g, const agpm_plan* plan, uint64_t seed, uint64_t first_id,
                 uint64_t count, double* values, uint8_t* hits, uint32_t* bindings, void* stream);
/* run_fixed_budget (ns_engine.cpp:142-153) */
int agpm_ns_fixed_budget(agpm_graph* g, const agpm_plan* plan, uint64_t budget, uint64_t seed,
                         agpm_accumulator* out, void* stream);
/* run_ns_online (ns_engine.cpp:106-140), workers=1 window semantics */
int agpm_ns_online(agpm_graph* g, const agpm_plan* plan, double eps, double delta,
                   const agpm_online_policy* policy, uint64_t seed, agpm_online_result* out,
                   void* stream);

/* Sampler strategy: 0 = auto (default), 1 = one warp per sample
 * (k-ary searches + coalesced chunk intersections), 2 = one lane per sample
 * (tiny adjacency lists), 3 = frontier phases (element-parallel
 * intersections over a whole batch), 5 = flat (a warp owns 32 samples, state on chip; each multi-list step
 * intersects the concatenation of the pending samples' drivers element-parallel,
 * picks lane-parallel). All strategies draw identical samples. (4, a fused
 * warp-per-sample-group sampler, was removed: slower than 3 and 5 everywhere.) */
int agpm_ns_set_strategy(int strategy);
/* The strategy a sampling launch of `count` ids of `plan` on `g` would run with
 * the current setting (the auto decision when the setting is 0): one of 1, 2, 3, 5. */
int agpm_ns_strategy_for(const agpm_graph* g, const agpm_plan* plan, uint64_t count, int* out_strategy);
/* Per-sample stream policy: 0 = CounterRng(seed, 0, sample_id) (default; the
 * reference's stream, bit-exact with its draw_sample), 1 = Philox4x32-10 keyed by
 * the seed with counter (draw index, sample id) — a counter-based stream of the
 * same (seed, id) addressing; eager plans on the flat sampler only (other
 * strategies raise AGPM_E_INVALID). */
int agpm_ns_set_rng(int policy);
/* frontier only: let a step whose lists nest the previous step's (cliques)
 * intersect that step's survivors instead of recomputing (same samples). */
int agpm_ns_set_frontier_reuse(int on);
/* flat and frontier samplers: dimension C of the dense-core adjacency bit matrix
 * (top C ids, C*C/8 bytes) that answers core-core membership tests in one
 * load; 0 disables; 0xffffffff = auto (default: 65536 up to 2^21 vertices,
 * 262144 up to 2^25, 524288 above, when it fits); at most 1048576. Results are
 * identical either way. */
int agpm_ns_set_core_dim(uint32_t dim);

/* Device-pointer building blocks (bench / multi-rank driver): enqueue only.
 * d_values: count f64 device buffer. */
int agpm_ns_sample_dev(agpm_graph* g, const agpm_plan* plan, uint64_t seed, uint64_t first_id,
                       uint64_t count, double* d_values, void* stream);
/* per-window moments (n, hits, sum, squared_sum) of d_values; windows of
 * `window` samples aligned to d_values[0]; out = ceil(count/window) entries */
int agpm_window_moments_dev(const double* d_values, uint64_t count, uint64_t window,
                            agpm_accumulator* d_out, void* stream);
/* Algorithmic bytes (SURVEY §8(d) B_min sector model) of ids [first, first+count),
 * summed on device: a counting replay of the same sample paths. */
int agpm_ns_bmin_bytes(agpm_graph* g, const agpm_plan* plan, uint64_t seed, uint64_t first_id,
                       uint64_t count, uint64_t* total_bytes, void* stream);

/* ------------------------------------------------- exact counting ---------
 * exact_count (exact_engine.cpp:66-91) for eager plans: oriented clique views
 * skip the order bounds (every arc is a seed), symmetric views apply them and
 * skip u > v seeds when the plan orients the seed edge. */
int agpm_exact_count(agpm_graph* g, const agpm_plan* plan, uint64_t* count, void* stream);
/* One shard of agpm_exact_count for multi-GPU counting: shard r of
 * nshards counts the seeds of 32-arc chunks r, r + nshards, ... (interleaved
 * over the arc array, so hub-heavy ranges spread over the ranks); the shards'
 * counts sum to agpm_exact_count. Ranks all-reduce the u64 partial counts. */
int agpm_exact_count_shard(agpm_graph* g, const agpm_plan* plan, uint32_t shard, uint32_t nshards,
                           uint64_t* count, void* stream);

/* ------------------------------------------- sparsification and GS -------
 * colour split: ColoredCsr::color_vertices (colored_csr.cpp:48-54) -> the
 *   zero-copy same-colour view (begin = offsets, end = split ends, colored_csr.cpp:90-93);
 *   colors_out (nullable, host) receives the n vertex colours.
 * Bernoulli: bernoulli_sparsify (csr_graph.cpp:190-213), a new plain CSR.
 * gs_estimate (gs_engine.cpp:42-75): scheme 0 = Bernoulli edge (scale p^-l),
 *   1 = colour (scale c^(k-1)); raw count from agpm_exact_count. */
typedef struct agpm_gs_result {
  double estimate;
  uint64_t raw_count;
  double scale;
  double preprocess_seconds, search_seconds;
} agpm_gs_result;

int agpm_color_split(agpm_graph* g, uint32_t colors, uint64_t seed, uint32_t* colors_out, uint64_t* same_edges,
                     agpm_graph** out, void* stream);
int agpm_bernoulli_sparsify(agpm_graph* g, double keep_probability, uint64_t seed, agpm_graph** out,
                            void* stream);
/* ColoredCsr::with_colors (colored_csr.cpp:14-46): colour split of the ORIGINAL
 * graph g for an explicit host colour array (every colour < color_count). */
int agpm_color_split_with_colors(agpm_graph* g, const uint32_t* colors, uint32_t color_count, uint64_t* same_edges,
                                 agpm_graph** out, void* stream);
/* ColoredCsr::merge_colors (colored_csr.cpp:56-88): coarsen the colouring
 * `colors` of the ORIGINAL graph g by group_map (length color_count, surjective
 * onto a contiguous [0, c')); coarse_out (nullable, host) receives the n coarse
 * colours. Errors: the reference's std::invalid_argument cases -> AGPM_E_INVALID. */
int agpm_merge_colors(agpm_graph* g, const uint32_t* colors, uint32_t color_count, const uint32_t* group_map,
                      uint32_t map_len, uint32_t* coarse_out, uint64_t* same_edges, agpm_graph** out,
                      void* stream);
int agpm_gs_estimate(agpm_graph* g, const agpm_plan* plan, int scheme, double keep_probability, uint32_t colors,
                     uint64_t seed, agpm_gs_result* out, void* stream);
/* triangle_count (csr_graph.cpp:225-239) */
int agpm_triangle_count(agpm_graph* g, uint64_t* count, void* stream);

/* --------------------------------------------- hybrid scheme choice -------
 * keep probability (gs_engine.cpp:24-40), NS cost cone (cost_model.cpp:78-110),
 * GS cost model (:112-145), fast profiler (:147-190, on device), selector
 * (:192-194), gamma probing (gs_engine.cpp:179-197 + exact_engine.cpp:135-213,
 * host), and the CLI's loose-mode orchestration (agpm_main.cpp:221-287). */
typedef struct agpm_keep_probability {
  double p;
  int32_t sparsification_useless;
  uint32_t color_count; /* floor(1/p), >= 1 */
} agpm_keep_probability;

typedef struct agpm_cost_cone {
  double lower_slope, upper_slope;
  uint64_t n_samples;
  double lower_time, upper_time;
} agpm_cost_cone;

typedef struct agpm_gs_cost {
  double preprocess_work, search_work, total_seconds;
  uint32_t color_count;
} agpm_gs_cost;

typedef struct agpm_profile_result {
  double n_samples_estimate, mu_prime, scaled_count, epsilon_hat_final;
  uint64_t n_converged;
  double fraction;
  int32_t reliable;
  double seconds;
} agpm_profile_result;

typedef struct agpm_hybrid_result {
  int32_t decision; /* 0 = NS (strict), 1 = GS */
  double estimate;
  double gamma;
  agpm_profile_result profile;
  agpm_keep_probability keep;
  agpm_cost_cone cone;
  agpm_gs_cost gs_model;
  agpm_gs_result gs;
  agpm_online_result ns;
} agpm_hybrid_result;

int agpm_choose_keep_probability(double eps, double delta, double count_estimate, double gamma_estimate,
                                 agpm_keep_probability* out);
int agpm_ns_cost_cone(double vertex_count, double arc_count, const agpm_plan* plan, uint64_t n_samples,
                      double hw_const, agpm_cost_cone* out);
int agpm_gs_cost_estimate(double vertex_count, double edge_count, const agpm_plan* plan, uint32_t colors,
                          double hw_const, uint64_t triangle_count, agpm_gs_cost* out);
int agpm_select_scheme(const agpm_cost_cone* cone, const agpm_gs_cost* gs); /* 1 = GS */
int agpm_count_matches_through_edge(const agpm_host_graph* g, const agpm_plan* plan, uint32_t u, uint32_t v,
                                    uint64_t* out);
int agpm_estimate_gamma(const agpm_host_graph* g, const agpm_plan* plan, uint64_t probe_edges, uint64_t seed,
                        int64_t work_budget, uint64_t* out);
/* brute_force_count (exact_engine.cpp:93-133): injective maps honouring the
 * induced mode / |Aut|, independent of the plan machinery; small graphs */
int agpm_brute_force_count(uint32_t n, const uint64_t* begin, const uint64_t* end, const uint32_t* neighbors,
                           const agpm_plan* plan, uint64_t* out);
/* the same two on a host CsrView (begin/end per vertex; end NULL = plain), with the
 * reference's optional in/out work budget (exact_engine.hpp:29-33, gs_engine.hpp:56-60) */
int agpm_count_matches_through_edge_view(uint32_t n, uint64_t edge_count, const uint64_t* begin,
                                         const uint64_t* end, const uint32_t* neighbors, const agpm_plan* plan,
                                         uint32_t u, uint32_t v, int64_t* work_budget, uint64_t* out);
int agpm_estimate_gamma_view(uint32_t n, uint64_t edge_count, const uint64_t* begin, const uint64_t* end,
                             const uint32_t* neighbors, const agpm_plan* plan, uint64_t probe_edges, uint64_t seed,
                             int64_t work_budget, uint64_t* out);
int agpm_fast_profile(agpm_graph* g, const agpm_plan* plan, double profile_fraction, double user_epsilon,
                      uint64_t seed, uint64_t profiler_sample_cap, agpm_profile_result* out, void* stream);
/* device analogue of calibrate_hardware_constant (cost_model.cpp:31-76): seconds
 * per cone work unit of the device sampler on a synthetic graph */
int agpm_calibrate_hardware_constant(double* out);
int agpm_count_hybrid(const agpm_host_graph* hg, agpm_graph* g, const agpm_plan* plan, double eps, double confidence,
                      uint64_t seed, double profile_fraction, double hw_const, agpm_hybrid_result* out, void* stream);

/* ---------------------------------------- dense/sparse region split -------
 * Builder-defined (no reference implementation). On a
 * degree-relabelled view: V_s = {deg < tau} = ids [0, tau_id); C_sparse =
 * matches touching V_s, exact; C_dense on G[V_d] by dense_method 0 = online NS
 * (eps, delta, max_samples), 1 = colour GS with `colors` colours repeated to
 * eps@delta (agpm_gs_online, at most `repeats` colourings; dense_ns holds that
 * run: windows = colourings), 2 = exact. estimate = C_sparse + C_dense. On an oriented clique DAG
 * tau_degree is taken as the id threshold tau_id itself. */
typedef struct agpm_region_result {
  uint32_t tau_id;
  uint32_t pad;
  uint64_t sparse_vertices, dense_vertices, dense_edges;
  int32_t rooted;      /* 1: C_sparse = root-restricted exact count; 0: exact(G) - exact(G[V_d]) */
  int32_t dense_exact; /* 1: C_dense is exact (method 2 or an empty dense region) */
  uint64_t c_sparse;
  double c_dense, estimate, dense_epsilon_hat;
  agpm_online_result dense_ns;
  double sparse_seconds, dense_seconds;
} agpm_region_result;

/* Colour-sparsified GS to a relative error bound: colouring
 * i (seed derive_key(seed, i, 0), `colors` colours) is one unbiased coarse sample
 * c^(k-1) x raw_i; the online detector (stats.cpp:57-70) stops at the first i >= 2
 * with eps_hat <= eps, else after max_colorings. out->windows = colourings run;
 * report / accumulator as for agpm_ns_online (sum over the X_i). */
int agpm_gs_online(agpm_graph* g, const agpm_plan* plan, uint32_t colors, double eps, double delta,
                   uint64_t max_colorings, uint64_t seed, agpm_online_result* out, void* stream);
/* exact count restricted to seeds whose first vertex is < root_limit */
int agpm_exact_count_rooted(agpm_graph* g, const agpm_plan* plan, uint32_t root_limit, uint64_t* count,
                            void* stream);
/* subgraph induced on vertices >= min_vertex (ids unchanged) */
int agpm_induced_suffix(agpm_graph* g, uint32_t min_vertex, agpm_graph** out, void* stream);
int agpm_region_split(agpm_graph* g, const agpm_plan* plan, uint32_t tau_degree, int dense_method, double eps,
                      double delta, uint64_t seed, uint32_t colors, uint32_t repeats, uint64_t max_samples,
                      agpm_region_result* out, void* stream);

/* ------------------------------------------------------- multi-GPU -------
 * SURVEY §8(e). The reference fans a window out over `workers` threads and
 * merges their accumulators in worker order (ns_engine.cpp:64-88, 121-137);
 * here a rank is one GPU holding a full replica of the view, global sample ids
 * are dealt to ranks in per-batch blocks (batch b, rank r: ids
 * [L_b + r*B, L_b + (r+1)*B)), each rank folds its block into window moments,
 * and the 32-B window records are all-gathered — rank order is id order, so
 * every rank runs the single-GPU stop test (converge_kernel) on the same
 * records and reaches the same decision: stop n, hits and sums equal the
 * single-GPU (= reference workers=1) run for every rank count.
 *
 * Communicators: NCCL (one process per GPU; rank 0 calls agpm_nccl_unique_id
 * and the caller broadcasts the 128 bytes), or a local group of `world` ranks
 * driven by host threads of one process (one thread per GPU; several ranks may
 * share a GPU — exchanges are host-synchronised peer copies, no kernel waits on
 * another rank). Create the communicator on the rank's device (cudaSetDevice
 * or agpm_set_device first). */
#define AGPM_NCCL_ID_BYTES 128
typedef struct agpm_comm agpm_comm;
typedef struct agpm_comm_group agpm_comm_group;
int agpm_nccl_unique_id(unsigned char id[AGPM_NCCL_ID_BYTES]);
int agpm_comm_init_nccl(int rank, int world, const unsigned char id[AGPM_NCCL_ID_BYTES], agpm_comm** out);
int agpm_comm_group_create(int world, agpm_comm_group** out);
int agpm_comm_init_local(agpm_comm_group* group, int rank, agpm_comm** out);
int agpm_comm_group_free(agpm_comm_group* group); /* after every member's agpm_comm_free */
int agpm_comm_free(agpm_comm* c);
int agpm_comm_info(const agpm_comm* c, int* rank, int* world, int* device, int* is_nccl);
/* enqueue an all-gather of device buffers on `stream`: d_recv[r*bytes ..] = rank r's d_send
 * (the exchange step of the sharded drivers, exposed for callers that drive
 * agpm_ns_sample_dev / agpm_window_moments_dev themselves) */
int agpm_comm_all_gather_dev(agpm_comm* c, const void* d_send, void* d_recv, uint64_t bytes_per_rank, void* stream);
/* run_ns_online (ns_engine.cpp:106-140) over the ranks of `c`; every rank
 * passes its own replica `g` and receives the same result (samples_launched
 * and seconds are global / this rank's). */
int agpm_ns_online_sharded(agpm_comm* c, agpm_graph* g, const agpm_plan* plan, double eps, double delta,
                           const agpm_online_policy* policy, uint64_t seed, agpm_online_result* out,
                           void* stream);
/* The id partition agpm_ns_online_sharded uses (host arithmetic, no device):
 * round of `launched` ids so far, per-rank block `batch` (a multiple of
 * `window`) -> this rank's first id / count, the round's id count, the number
 * of valid (id-ordered, prefix) window records in the gather and the records
 * each rank contributes. Exposed so multi-rank host logic can be tested on CPU. */
typedef struct agpm_shard_round {
  uint64_t first_id, count, round_ids, valid_windows, windows_per_rank;
} agpm_shard_round;
int agpm_ns_shard_round(uint64_t launched, uint64_t batch, uint64_t window, uint64_t max_samples, int rank,
                        int world, agpm_shard_round* out);
/* run_fixed_budget (ns_engine.cpp:142-153) over the ranks: rank r draws the
 * r-th contiguous share of ids [0, budget); accumulators gathered and folded in
 * rank order (n, hits exact; sums equal up to reduction-order rounding). */
int agpm_ns_fixed_budget_sharded(agpm_comm* c, agpm_graph* g, const agpm_plan* plan, uint64_t budget,
                                 uint64_t seed, agpm_accumulator* out, void* stream);
/* exact_count (exact_engine.cpp:66-91) over the ranks (agpm_exact_count_shard
 * per rank, u64 partials summed) */
int agpm_exact_count_sharded(agpm_comm* c, agpm_graph* g, const agpm_plan* plan, uint64_t* count, void* stream);

/* ------------------------------------------------------- misc / device -----*/
const char* agpm_last_error(void);
int agpm_device_count(int* n);
int agpm_set_device(int device);
/* the calling thread's current CUDA device (-1 if none) */
int agpm_current_device(void);
int agpm_version(void);
int agpm_sync(void* stream);
/* kernels launched by this library since load (evidence for the bench) */
uint64_t agpm_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* AGPM_B200_H_ */
