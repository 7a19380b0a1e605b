"""ctypes image of include/agpm_b200.h (structs + prototypes).

Shared by the product binding (paper_2405_03488_b200/__init__.py) and the
test-only oracle bindings (tests/oracle_bindings.py), which pass the same
agpm_plan / agpm_accumulator layouts across their own C-ABIs.
"""
import ctypes as C

MAX_K = 9
MAX_PAIRS = 36

OK, E_INVALID, E_PATTERN, E_IO, E_PARSE, E_CUDA, E_NODEVICE, E_INTERNAL = range(8)

Pairs = (C.c_int32 * 2) * MAX_PAIRS


class PlanStep(C.Structure):
    _fields_ = [
        ("pattern_vertex", C.c_int32),
        ("n_in", C.c_int32), ("in_positions", C.c_int32 * MAX_K),
        ("n_out", C.c_int32), ("out_positions", C.c_int32 * MAX_K),
        ("n_gt", C.c_int32), ("greater_than", C.c_int32 * MAX_K),
        ("n_lt", C.c_int32), ("less_than", C.c_int32 * MAX_K),
        ("tree_parent", C.c_int32),
        ("n_verify", C.c_int32), ("verify_edges", (C.c_int32 * 2) * MAX_K),
    ]


class Plan(C.Structure):
    _fields_ = [
        ("name", C.c_char * 64),
        ("k", C.c_int32),
        ("induced", C.c_int32),
        ("n_edges", C.c_int32), ("edges", Pairs),
        ("adjacency", C.c_uint32 * MAX_K),
        ("verify_mode", C.c_int32),
        ("order", C.c_int32 * MAX_K), ("pos_of", C.c_int32 * MAX_K),
        ("seed_ordered", C.c_int32), ("symmetry_enabled", C.c_int32),
        ("n_steps", C.c_int32),
        ("steps", PlanStep * (MAX_K - 2)),
        ("n_closure", C.c_int32), ("closure_edges", Pairs),
        ("n_constraints", C.c_int32), ("constraints", Pairs),
        ("n_terminal", C.c_int32), ("terminal_constraints", Pairs),
    ]

    def to_dict(self):
        """Reference-shaped view (plan.hpp:21-55) used by the plan parity tests."""
        def pairs(n, arr):
            return [[arr[i][0], arr[i][1]] for i in range(n)]

        steps = []
        for s in range(self.n_steps):
            st = self.steps[s]
            steps.append({
                "pattern_vertex": st.pattern_vertex,
                "in_positions": list(st.in_positions[: st.n_in]),
                "out_positions": list(st.out_positions[: st.n_out]),
                "greater_than": list(st.greater_than[: st.n_gt]),
                "less_than": list(st.less_than[: st.n_lt]),
                "tree_parent": st.tree_parent,
                "verify_edges": [[st.verify_edges[i][0], st.verify_edges[i][1]] for i in range(st.n_verify)],
            })
        return {
            "name": self.name.decode(),
            "k": self.k,
            "induced": self.induced,
            "edges": pairs(self.n_edges, self.edges),
            "adjacency": list(self.adjacency[: self.k]),
            "verify_mode": self.verify_mode,
            "order": list(self.order[: self.k]),
            "pos_of": list(self.pos_of[: self.k]),
            "seed_ordered": self.seed_ordered,
            "symmetry_enabled": self.symmetry_enabled,
            "steps": steps,
            "closure_edges": pairs(self.n_closure, self.closure_edges),
            "constraints": pairs(self.n_constraints, self.constraints),
            "terminal_constraints": pairs(self.n_terminal, self.terminal_constraints),
        }


class Accumulator(C.Structure):
    _fields_ = [("n", C.c_uint64), ("hits", C.c_uint64), ("sum", C.c_double), ("squared_sum", C.c_double)]

    def add(self, value, hit):  # stats.hpp:22-27
        self.n += 1
        self.hits += 1 if hit else 0
        self.sum += value
        self.squared_sum += value * value

    def merge(self, o):  # stats.hpp:28-33
        self.n += o.n
        self.hits += o.hits
        self.sum += o.sum
        self.squared_sum += o.squared_sum


class Report(C.Structure):
    _fields_ = [("mu", C.c_double), ("sigma", C.c_double), ("epsilon_hat", C.c_double), ("n", C.c_uint64),
                ("converged", C.c_int32), ("hit_rate", C.c_double)]


class OnlinePolicy(C.Structure):
    _fields_ = [("n_min", C.c_uint64), ("max_samples", C.c_uint64), ("profiled_n_samples", C.c_uint64)]

    def __init__(self, n_min=1000, max_samples=1000000000, profiled_n_samples=0):
        super().__init__(n_min, max_samples, profiled_n_samples)


class OnlineResult(C.Structure):
    _fields_ = [("report", Report), ("accumulator", Accumulator), ("windows", C.c_uint64),
                ("work_units", C.c_uint64), ("samples_launched", C.c_uint64), ("seconds", C.c_double)]


class GsResult(C.Structure):
    _fields_ = [("estimate", C.c_double), ("raw_count", C.c_uint64), ("scale", C.c_double),
                ("preprocess_seconds", C.c_double), ("search_seconds", C.c_double)]


class KeepProbability(C.Structure):
    _fields_ = [("p", C.c_double), ("sparsification_useless", C.c_int32), ("color_count", C.c_uint32)]


class CostCone(C.Structure):
    _fields_ = [("lower_slope", C.c_double), ("upper_slope", C.c_double), ("n_samples", C.c_uint64),
                ("lower_time", C.c_double), ("upper_time", C.c_double)]


class GsCost(C.Structure):
    _fields_ = [("preprocess_work", C.c_double), ("search_work", C.c_double), ("total_seconds", C.c_double),
                ("color_count", C.c_uint32)]


class ProfileResult(C.Structure):
    _fields_ = [("n_samples_estimate", C.c_double), ("mu_prime", C.c_double), ("scaled_count", C.c_double),
                ("epsilon_hat_final", C.c_double), ("n_converged", C.c_uint64), ("fraction", C.c_double),
                ("reliable", C.c_int32), ("seconds", C.c_double)]


class HybridResult(C.Structure):
    _fields_ = [("decision", C.c_int32), ("estimate", C.c_double), ("gamma", C.c_double),
                ("profile", ProfileResult), ("keep", KeepProbability), ("cone", CostCone), ("gs_model", GsCost),
                ("gs", GsResult), ("ns", OnlineResult)]


class RegionResult(C.Structure):
    _fields_ = [("tau_id", C.c_uint32), ("pad", C.c_uint32), ("sparse_vertices", C.c_uint64),
                ("dense_vertices", C.c_uint64), ("dense_edges", C.c_uint64), ("rooted", C.c_int32),
                ("dense_exact", C.c_int32), ("c_sparse", C.c_uint64), ("c_dense", C.c_double),
                ("estimate", C.c_double), ("dense_epsilon_hat", C.c_double), ("dense_ns", OnlineResult),
                ("sparse_seconds", C.c_double), ("dense_seconds", C.c_double)]


P = C.c_void_p
u32, u64, i32, dbl = C.c_uint32, C.c_uint64, C.c_int, C.c_double
pu32, pu64, pdbl, pu8 = C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), C.POINTER(C.c_double), C.POINTER(C.c_uint8)
pPlan, pAcc = C.POINTER(Plan), C.POINTER(Accumulator)


class ShardRound(C.Structure):
    """agpm_shard_round: this rank's ids in one round of the sharded online loop."""
    _fields_ = [("first_id", C.c_uint64), ("count", C.c_uint64), ("round_ids", C.c_uint64),
                ("valid_windows", C.c_uint64), ("windows_per_rank", C.c_uint64)]


NCCL_ID_BYTES = 128
