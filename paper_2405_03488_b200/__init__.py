"""B200-native ScaleGPM sampling hot path — Python mirror of the reference API.

The product is libagpm_b200.so (host C++ + sm_100a kernels behind the C-ABI in
include/agpm_b200.h). This module binds it with ctypes and mirrors the
reference's agpm:: names and semantics (csr_graph.hpp, pattern.hpp, plan.hpp,
stats.hpp, ns_engine.hpp) so callers and tests read like the reference's own:

    g = CsrGraph.load("graph.bin")             # load_graph_auto
    plan = compile_plan("4clique", "eager")   # parse_pattern_spec + compile_plan
    dg = DeviceGraph(g)                        # device-resident CsrView
    res = run_ns_online(dg, plan, 0.01, 0.05, OnlinePolicy(), seed=1)

There is no CPU fallback: if the shared library is missing or no CUDA device
is visible, calls raise (ExtensionMissing / NoDeviceError).
"""
import ctypes as C
import os

import numpy as np

from . import _abi
from ._abi import Accumulator, OnlinePolicy, OnlineResult, Plan, Report

__all__ = [
    "AgpmError", "PatternError", "IoError", "ParseError", "CudaError", "NoDeviceError", "ExtensionMissing",
    "lib", "compile_plan", "builtin_pattern_names", "automorphism_count", "scaling_rule_text",
    "plan_verifies_each_edge_once", "norm_cdf", "inv_norm_cdf", "predicted_error", "CsrGraph",
    "er_graph", "er_fast", "rmat", "DeviceGraph", "draw_samples", "run_fixed_budget", "run_ns_online",
    "hit_rate_report", "exact_count", "exact_count_rooted", "region_split", "gs_estimate", "choose_keep_probability", "ns_cost_cone",
    "gs_cost_estimate", "select_scheme", "count_matches_through_edge", "estimate_gamma", "fast_profile",
    "calibrate_hardware_constant", "count_hybrid", "exact_count_shard", "gs_online", "bmin_bytes", "set_strategy", "strategy_for", "set_rng", "sample_dev", "window_moments_dev", "kernel_launches", "device_count",
    "Comm", "LocalGroup", "nccl_unique_id", "shard_round", "run_ns_online_sharded", "run_fixed_budget_sharded",
    "exact_count_sharded",
    "Accumulator", "OnlinePolicy", "OnlineResult", "Plan", "Report", "LIB_PATH",
]

# AGPM_LIB: a side build of the same sources (csrc/Makefile SUFFIX=...) for A/B timing
LIB_PATH = os.environ.get("AGPM_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libagpm_b200.so")


class AgpmError(RuntimeError):
    pass


class PatternError(AgpmError):  # agpm::pattern_error (pattern.hpp:49-51)
    pass


class IoError(AgpmError):  # agpm::io_error (csr_graph.hpp:15-17)
    pass


class ParseError(AgpmError):  # agpm::parse_error (csr_graph.hpp:12-14)
    pass


class CudaError(AgpmError):
    pass


class NoDeviceError(AgpmError):
    pass


class ExtensionMissing(ImportError):
    pass


_lib = None


def lib():
    """Load libagpm_b200.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ExtensionMissing(f"{LIB_PATH} is not built (run __graft_entry__.build()); "
                                   "the sampling path has no CPU fallback")
        L = C.CDLL(LIB_PATH)
        _declare(L)
        _lib = L
    return _lib


def _declare(L):
    A = _abi
    sig = {
        "agpm_last_error": (C.c_char_p, []),
        "agpm_version": (C.c_int, []),
        "agpm_kernel_launches": (A.u64, []),
        "agpm_device_count": (C.c_int, [C.POINTER(C.c_int)]),
        "agpm_set_device": (C.c_int, [C.c_int]),
        "agpm_sync": (C.c_int, [A.P]),
        "agpm_plan_compile": (C.c_int, [C.c_char_p, C.c_char_p, C.c_int, C.c_int, A.pPlan]),
        "agpm_builtin_pattern_names": (C.c_int, [C.c_char_p, C.c_size_t]),
        "agpm_pattern_automorphism_count": (C.c_int, [C.c_char_p, C.c_char_p, A.pu64]),
        "agpm_plan_scaling_rule": (C.c_int, [A.pPlan, C.c_char_p, C.c_size_t]),
        "agpm_plan_verifies_each_edge_once": (C.c_int, [A.pPlan, C.POINTER(C.c_int)]),
        "agpm_norm_cdf": (C.c_double, [C.c_double]),
        "agpm_inv_norm_cdf": (C.c_int, [C.c_double, A.pdbl]),
        "agpm_predicted_error": (C.c_int, [A.pAcc, C.c_double, C.POINTER(Report)]),
        "agpm_host_graph_from_edges": (C.c_int, [A.pu32, A.u64, A.u32, C.POINTER(A.P)]),
        "agpm_host_graph_from_csr": (C.c_int, [A.u32, A.u64, A.pu64, A.pu32, C.c_int, C.POINTER(A.P)]),
        "agpm_host_graph_load": (C.c_int, [C.c_char_p, C.POINTER(A.P)]),
        "agpm_host_graph_write_binary": (C.c_int, [A.P, C.c_char_p]),
        "agpm_host_graph_info": (C.c_int, [A.P, A.pu32, A.pu64, A.pu64, C.POINTER(C.c_int), A.pu64]),
        "agpm_host_graph_arrays": (C.c_int, [A.P, C.POINTER(A.pu64), C.POINTER(A.pu32)]),
        "agpm_host_graph_free": (None, [A.P]),
        "agpm_host_graph_relabel_by_degree": (C.c_int, [A.P, C.POINTER(A.P)]),
        "agpm_host_graph_orient_by_degree": (C.c_int, [A.P, C.POINTER(A.P)]),
        "agpm_gen_er_pairs": (C.c_int, [A.u32, C.c_double, A.u64, C.POINTER(A.P)]),
        "agpm_gen_er_fast": (C.c_int, [A.u32, A.u64, A.u64, A.u32, A.u32, C.POINTER(A.P)]),
        "agpm_gen_rmat": (C.c_int, [A.u32, A.u32, C.c_double, C.c_double, C.c_double, A.u64, C.POINTER(A.P)]),
        "agpm_graph_upload": (C.c_int, [A.u32, A.u64, A.pu64, A.pu64, A.pu32, A.u64, C.c_int, A.P, C.POINTER(A.P)]),
        "agpm_graph_upload_host": (C.c_int, [A.P, A.P, C.POINTER(A.P)]),
        "agpm_graph_prepare": (C.c_int, [A.P, A.P]),
        "agpm_host_graph_pin": (C.c_int, [A.P]),
        "agpm_graph_free": (C.c_int, [A.P]),
        "agpm_graph_info": (C.c_int, [A.P, A.pu32, A.pu64, A.pu64, C.POINTER(C.c_int), A.pu64]),
        "agpm_graph_download": (C.c_int, [A.P, A.pu64, A.pu64, A.pu32]),
        "agpm_graph_neighbor_len": (C.c_int, [A.P, A.pu64]),
        "agpm_graph_from_edges_device": (C.c_int, [A.pu32, A.u64, A.u32, C.c_int, A.P, C.POINTER(A.P)]),
        "agpm_gen_rmat_device": (C.c_int, [A.u32, A.u32, C.c_double, C.c_double, C.c_double, A.u64, C.c_int, A.P,
                                           C.POINTER(A.P)]),
        "agpm_gen_er_fast_device": (C.c_int, [A.u32, A.u64, A.u64, A.u32, A.u32, C.c_int, A.P, C.POINTER(A.P)]),
        "agpm_graph_relabel_device": (C.c_int, [A.P, A.P, C.POINTER(A.P)]),
        "agpm_graph_orient_device": (C.c_int, [A.P, A.P, C.POINTER(A.P)]),
        "agpm_ns_draw": (C.c_int, [A.P, A.pPlan, A.u64, A.u64, A.u64, A.pdbl, A.pu8, A.pu32, A.P]),
        "agpm_ns_fixed_budget": (C.c_int, [A.P, A.pPlan, A.u64, A.u64, A.pAcc, A.P]),
        "agpm_ns_online": (C.c_int, [A.P, A.pPlan, C.c_double, C.c_double, C.POINTER(OnlinePolicy), A.u64,
                                     C.POINTER(OnlineResult), A.P]),
        "agpm_ns_sample_dev": (C.c_int, [A.P, A.pPlan, A.u64, A.u64, A.u64, A.P, A.P]),
        "agpm_window_moments_dev": (C.c_int, [A.P, A.u64, A.u64, A.P, A.P]),
        "agpm_ns_bmin_bytes": (C.c_int, [A.P, A.pPlan, A.u64, A.u64, A.u64, A.pu64, A.P]),
        "agpm_ns_set_strategy": (C.c_int, [C.c_int]),
        "agpm_ns_strategy_for": (C.c_int, [A.P, A.pPlan, A.u64, C.POINTER(C.c_int)]),
        "agpm_exact_count": (C.c_int, [A.P, A.pPlan, A.pu64, A.P]),
        "agpm_exact_count_shard": (C.c_int, [A.P, A.pPlan, A.u32, A.u32, A.pu64, A.P]),
        "agpm_gs_online": (C.c_int, [A.P, A.pPlan, A.u32, C.c_double, C.c_double, A.u64, A.u64,
                                     C.POINTER(A.OnlineResult), A.P]),
        "agpm_color_split_with_colors": (C.c_int, [A.P, A.pu32, A.u32, A.pu64, C.POINTER(A.P), A.P]),
        "agpm_merge_colors": (C.c_int, [A.P, A.pu32, A.u32, A.pu32, A.u32, A.pu32, A.pu64, C.POINTER(A.P), A.P]),
        "agpm_color_split": (C.c_int, [A.P, A.u32, A.u64, A.pu32, A.pu64, C.POINTER(A.P), A.P]),
        "agpm_bernoulli_sparsify": (C.c_int, [A.P, C.c_double, A.u64, C.POINTER(A.P), A.P]),
        "agpm_gs_estimate": (C.c_int, [A.P, A.pPlan, C.c_int, C.c_double, A.u32, A.u64, C.POINTER(A.GsResult), A.P]),
        "agpm_triangle_count": (C.c_int, [A.P, A.pu64, A.P]),
        "agpm_graph_max_degree": (C.c_int, [A.P, A.pu64]),
        "agpm_exact_count_rooted": (C.c_int, [A.P, A.pPlan, A.u32, A.pu64, A.P]),
        "agpm_induced_suffix": (C.c_int, [A.P, A.u32, C.POINTER(A.P), A.P]),
        "agpm_region_split": (C.c_int, [A.P, A.pPlan, A.u32, C.c_int, C.c_double, C.c_double, A.u64, A.u32, A.u32,
                                        A.u64, C.POINTER(A.RegionResult), A.P]),
        "agpm_choose_keep_probability": (C.c_int, [C.c_double] * 4 + [C.POINTER(A.KeepProbability)]),
        "agpm_ns_cost_cone": (C.c_int, [C.c_double, C.c_double, A.pPlan, A.u64, C.c_double, C.POINTER(A.CostCone)]),
        "agpm_gs_cost_estimate": (C.c_int, [C.c_double, C.c_double, A.pPlan, A.u32, C.c_double, A.u64,
                                            C.POINTER(A.GsCost)]),
        "agpm_select_scheme": (C.c_int, [C.POINTER(A.CostCone), C.POINTER(A.GsCost)]),
        "agpm_count_matches_through_edge": (C.c_int, [A.P, A.pPlan, A.u32, A.u32, A.pu64]),
        "agpm_estimate_gamma": (C.c_int, [A.P, A.pPlan, A.u64, A.u64, C.c_int64, A.pu64]),
        "agpm_fast_profile": (C.c_int, [A.P, A.pPlan, C.c_double, C.c_double, A.u64, A.u64,
                                        C.POINTER(A.ProfileResult), A.P]),
        "agpm_calibrate_hardware_constant": (C.c_int, [A.pdbl]),
        "agpm_count_hybrid": (C.c_int, [A.P, A.P, A.pPlan, C.c_double, C.c_double, A.u64, C.c_double, C.c_double,
                                        C.POINTER(A.HybridResult), A.P]),
        "agpm_ns_set_frontier_reuse": (C.c_int, [C.c_int]),
        "agpm_ns_set_core_dim": (C.c_int, [A.u32]),
        "agpm_ns_set_rng": (C.c_int, [C.c_int]),
        "agpm_nccl_unique_id": (C.c_int, [C.c_char_p]),
        "agpm_comm_init_nccl": (C.c_int, [C.c_int, C.c_int, C.c_char_p, C.POINTER(A.P)]),
        "agpm_comm_group_create": (C.c_int, [C.c_int, C.POINTER(A.P)]),
        "agpm_comm_init_local": (C.c_int, [A.P, C.c_int, C.POINTER(A.P)]),
        "agpm_comm_group_free": (C.c_int, [A.P]),
        "agpm_comm_free": (C.c_int, [A.P]),
        "agpm_comm_info": (C.c_int, [A.P] + [C.POINTER(C.c_int)] * 4),
        "agpm_ns_shard_round": (C.c_int, [A.u64, A.u64, A.u64, A.u64, C.c_int, C.c_int,
                                          C.POINTER(A.ShardRound)]),
        "agpm_ns_online_sharded": (C.c_int, [A.P, A.P, A.pPlan, C.c_double, C.c_double, C.POINTER(OnlinePolicy),
                                             A.u64, C.POINTER(OnlineResult), A.P]),
        "agpm_ns_fixed_budget_sharded": (C.c_int, [A.P, A.P, A.pPlan, A.u64, A.u64, A.pAcc, A.P]),
        "agpm_exact_count_sharded": (C.c_int, [A.P, A.P, A.pPlan, A.pu64, A.P]),
        "agpm_comm_all_gather_dev": (C.c_int, [A.P, A.P, A.P, A.u64, A.P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args


def _check(status):
    if status == _abi.OK:
        return
    msg = lib().agpm_last_error().decode(errors="replace")
    exc = {
        _abi.E_INVALID: ValueError,  # std::invalid_argument
        _abi.E_PATTERN: PatternError,
        _abi.E_IO: IoError,
        _abi.E_PARSE: ParseError,
        _abi.E_CUDA: CudaError,
        _abi.E_NODEVICE: NoDeviceError,
    }.get(status, AgpmError)
    raise exc(msg)


def _b(s):
    return s.encode() if isinstance(s, str) else (s or b"")


def _ptr(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


# ------------------------------------------------------------------ patterns / plans
_MODES = {"eager": 0, "lazy": 1, 0: 0, 1: 1}


def compile_plan(spec, mode="eager", enable_symmetry=True, induced=""):
    """parse_pattern_spec(spec, induced) + compile_plan(p, mode, enable_symmetry)
    (pattern.cpp:130-165, plan.cpp:57-137)."""
    plan = Plan()
    _check(lib().agpm_plan_compile(_b(spec), _b(induced), _MODES[mode], int(bool(enable_symmetry)),
                                   C.byref(plan)))
    return plan


def builtin_pattern_names():
    buf = C.create_string_buffer(4096)
    _check(lib().agpm_builtin_pattern_names(buf, 4096))
    return buf.value.decode().split()


def automorphism_count(spec, induced=""):
    out = C.c_uint64()
    _check(lib().agpm_pattern_automorphism_count(_b(spec), _b(induced), C.byref(out)))
    return out.value


def scaling_rule_text(plan):
    buf = C.create_string_buffer(512)
    _check(lib().agpm_plan_scaling_rule(C.byref(plan), buf, 512))
    return buf.value.decode()


def plan_verifies_each_edge_once(plan):
    out = C.c_int()
    _check(lib().agpm_plan_verifies_each_edge_once(C.byref(plan), C.byref(out)))
    return bool(out.value)


# ------------------------------------------------------------------ stats
def norm_cdf(z):
    return lib().agpm_norm_cdf(z)


def inv_norm_cdf(q):
    out = C.c_double()
    _check(lib().agpm_inv_norm_cdf(q, C.byref(out)))
    return out.value


def predicted_error(acc, delta):
    rep = Report()
    _check(lib().agpm_predicted_error(C.byref(acc), delta, C.byref(rep)))
    return rep


# ------------------------------------------------------------------ host graphs
class CsrGraph:
    """Owning host CSR (agpm::CsrGraph, csr_graph.hpp:46-80)."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value and _lib is not None:
            _lib.agpm_host_graph_free(h)
            self._h = None

    @staticmethod
    def _make(fn, *args):
        h = C.c_void_p()
        _check(fn(*args, C.byref(h)))
        return CsrGraph(h)

    @classmethod
    def from_edges(cls, edges, min_vertex_count=0):
        e = np.ascontiguousarray(np.asarray(edges, dtype=np.uint32).reshape(-1, 2))
        return cls._make(lib().agpm_host_graph_from_edges, _ptr(e, C.c_uint32), e.shape[0], min_vertex_count)

    @classmethod
    def from_csr(cls, offsets, neighbors, edge_count, oriented=False):
        o = np.ascontiguousarray(offsets, dtype=np.uint64)
        nb = np.ascontiguousarray(neighbors, dtype=np.uint32)
        return cls._make(lib().agpm_host_graph_from_csr, len(o) - 1, edge_count, _ptr(o, C.c_uint64),
                         _ptr(nb, C.c_uint32), int(oriented))

    @classmethod
    def load(cls, path):
        return cls._make(lib().agpm_host_graph_load, _b(path))

    def write_binary(self, path):
        _check(lib().agpm_host_graph_write_binary(self._h, _b(path)))

    def _info(self):
        n, m, arcs, o, md = C.c_uint32(), C.c_uint64(), C.c_uint64(), C.c_int(), C.c_uint64()
        _check(lib().agpm_host_graph_info(self._h, C.byref(n), C.byref(m), C.byref(arcs), C.byref(o), C.byref(md)))
        return n.value, m.value, arcs.value, bool(o.value), md.value

    @property
    def vertex_count(self):
        return self._info()[0]

    @property
    def edge_count(self):
        return self._info()[1]

    @property
    def arc_count(self):
        return self._info()[2]

    @property
    def oriented(self):
        return self._info()[3]

    def max_degree(self):
        return self._info()[4]

    def arrays(self):
        """(offsets u64[n+1], neighbors u32[arcs]) as numpy copies."""
        n, _, arcs, _, _ = self._info()
        po, pn = C.POINTER(C.c_uint64)(), C.POINTER(C.c_uint32)()
        _check(lib().agpm_host_graph_arrays(self._h, C.byref(po), C.byref(pn)))
        off = np.ctypeslib.as_array(po, shape=(n + 1,)).copy()
        nbr = np.ctypeslib.as_array(pn, shape=(arcs,)).copy() if arcs else np.zeros(0, np.uint32)
        return off, nbr

    def pin(self):
        """Page-lock the arrays (cudaHostRegister) so device uploads run at DMA speed."""
        _check(lib().agpm_host_graph_pin(self._h))
        return self

    def relabel_by_degree(self):
        return CsrGraph._make(lib().agpm_host_graph_relabel_by_degree, self._h)

    def orient_by_degree(self):
        return CsrGraph._make(lib().agpm_host_graph_orient_by_degree, self._h)


def er_graph(n, p, seed):
    """The reference's er_graph (test_graphs.hpp:37-43), multi-threaded."""
    return CsrGraph._make(lib().agpm_gen_er_pairs, n, p, seed)


def er_fast(n, target_edges, seed, planted_k=0, planted_count=0):
    return CsrGraph._make(lib().agpm_gen_er_fast, n, target_edges, seed, planted_k, planted_count)


def rmat(scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1):
    return CsrGraph._make(lib().agpm_gen_rmat, scale, edge_factor, a, b, c, seed)


# ------------------------------------------------------------------ device graphs
def _device_make(fn, *args):
    h = C.c_void_p()
    _check(fn(*args, C.byref(h)))
    return DeviceGraph(_handle=h)


def rmat_device(scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1, relabel=True, stream=None):
    """rmat(...)[.relabel_by_degree()] built in HBM (agpm_gen_rmat_device)."""
    return _device_make(lib().agpm_gen_rmat_device, scale, edge_factor, a, b, c, seed, int(relabel), stream)


def er_fast_device(n, target_edges, seed, planted_k=0, planted_count=0, relabel=True, stream=None):
    """er_fast(...)[.relabel_by_degree()] built in HBM (agpm_gen_er_fast_device)."""
    return _device_make(lib().agpm_gen_er_fast_device, n, target_edges, seed, planted_k, planted_count,
                        int(relabel), stream)


def graph_from_edges_device(pairs, min_vertex_count=0, relabel=False, stream=None):
    """CsrGraph::from_edges (csr_graph.cpp:46-72) built in HBM; pairs = (m, 2) ints."""
    p = np.ascontiguousarray(np.asarray(pairs, dtype=np.uint32).reshape(-1, 2))
    return _device_make(lib().agpm_graph_from_edges_device, _ptr(p, C.c_uint32), len(p), min_vertex_count,
                        int(relabel), stream)


class DeviceGraph:
    """Device-resident CsrView mirror (agpm_graph)."""

    def __init__(self, graph=None, *, begin=None, end=None, neighbors=None, vertex_count=None, edge_count=None,
                 oriented=False, stream=None, _handle=None):
        h = C.c_void_p()
        if _handle is not None:
            h = _handle
        elif graph is not None:
            _check(lib().agpm_graph_upload_host(graph._h, stream, C.byref(h)))
        else:
            b = np.ascontiguousarray(begin, dtype=np.uint64)
            e = None if end is None else np.ascontiguousarray(end, dtype=np.uint64)
            nb = np.ascontiguousarray(neighbors, dtype=np.uint32)
            n = vertex_count if vertex_count is not None else (len(b) - 1 if e is None else len(b))
            _check(lib().agpm_graph_upload(n, edge_count, _ptr(b, C.c_uint64),
                                           None if e is None else _ptr(e, C.c_uint64), _ptr(nb, C.c_uint32),
                                           len(nb), int(oriented), stream, C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value and _lib is not None:
            _lib.agpm_graph_free(h)
            self._h = None

    def prepare(self, stream=None):
        """Build the sampling indexes (dense core, twin arcs) now; same samples either way."""
        _check(lib().agpm_graph_prepare(self._h, stream))
        return self

    def relabel_by_degree(self, stream=None):
        """relabel_by_degree on the device (plain undirected views)."""
        return _device_make(lib().agpm_graph_relabel_device, self._h, stream)

    def orient_by_degree(self, stream=None):
        """orient_by_degree (csr_graph.cpp:172) on the device."""
        return _device_make(lib().agpm_graph_orient_device, self._h, stream)

    def download(self):
        """(begin u64[n], end u64[n], neighbors u32[neighbor_len]) of the view (tests)."""
        n = self.info()["vertex_count"]
        nl = C.c_uint64()
        _check(lib().agpm_graph_neighbor_len(self._h, C.byref(nl)))
        b = np.zeros(max(n, 1), np.uint64)
        e = np.zeros(max(n, 1), np.uint64)
        nb = np.zeros(max(nl.value, 1), np.uint32)
        _check(lib().agpm_graph_download(self._h, _ptr(b, C.c_uint64), _ptr(e, C.c_uint64), _ptr(nb, C.c_uint32)))
        return b[:n], e[:n], nb[: nl.value]

    def color_split(self, colors, seed, stream=None):
        """ColoredCsr::color_vertices -> (same-colour view, host colours, same-colour edge count)."""
        n = self.info()["vertex_count"]
        cols = np.zeros(max(n, 1), np.uint32)
        same = C.c_uint64()
        h = C.c_void_p()
        _check(lib().agpm_color_split(self._h, colors, seed, _ptr(cols, C.c_uint32), C.byref(same), C.byref(h), stream))
        return DeviceGraph(_handle=h), cols[:n], same.value

    def color_split_with_colors(self, colors, color_count, stream=None):
        """ColoredCsr::with_colors -> (same-colour view, same-colour edge count)."""
        cols = np.ascontiguousarray(colors, np.uint32)
        same = C.c_uint64()
        h = C.c_void_p()
        _check(lib().agpm_color_split_with_colors(self._h, _ptr(cols, C.c_uint32), color_count, C.byref(same),
                                                  C.byref(h), stream))
        return DeviceGraph(_handle=h), same.value

    def merge_colors(self, colors, color_count, group_map, stream=None):
        """ColoredCsr::merge_colors of the colouring `colors` (of this graph) by group_map ->
        (coarse same-colour view, coarse colours, same-colour edge count)."""
        cols = np.ascontiguousarray(colors, np.uint32)
        gm = np.ascontiguousarray(group_map, np.uint32)
        n = self.info()["vertex_count"]
        coarse = np.zeros(max(n, 1), np.uint32)
        same = C.c_uint64()
        h = C.c_void_p()
        _check(lib().agpm_merge_colors(self._h, _ptr(cols, C.c_uint32), color_count, _ptr(gm, C.c_uint32), len(gm),
                                       _ptr(coarse, C.c_uint32), C.byref(same), C.byref(h), stream))
        return DeviceGraph(_handle=h), coarse[:n], same.value

    def bernoulli_sparsify(self, keep_probability, seed, stream=None):
        h = C.c_void_p()
        _check(lib().agpm_bernoulli_sparsify(self._h, keep_probability, seed, C.byref(h), stream))
        return DeviceGraph(_handle=h)

    def induced_suffix(self, min_vertex, stream=None):
        """Subgraph induced on vertices >= min_vertex (the dense region of a relabelled graph)."""
        h = C.c_void_p()
        _check(lib().agpm_induced_suffix(self._h, min_vertex, C.byref(h), stream))
        return DeviceGraph(_handle=h)

    def triangle_count(self, stream=None):
        out = C.c_uint64()
        _check(lib().agpm_triangle_count(self._h, C.byref(out), stream))
        return out.value

    def info(self):
        n, m, arcs, o, by = C.c_uint32(), C.c_uint64(), C.c_uint64(), C.c_int(), C.c_uint64()
        _check(lib().agpm_graph_info(self._h, C.byref(n), C.byref(m), C.byref(arcs), C.byref(o), C.byref(by)))
        md = C.c_uint64()
        _check(lib().agpm_graph_max_degree(self._h, C.byref(md)))
        return {"vertex_count": n.value, "edge_count": m.value, "arcs": arcs.value, "oriented": bool(o.value),
                "device_bytes": by.value, "max_degree": md.value}


def draw_samples(dg, plan, seed, first_id, count, with_bindings=True, stream=None):
    """draw_sample for ids [first_id, first_id+count) with CounterRng(seed, 0, id)
    (ns_engine.cpp:92-104). Returns (values f64, hits u8, bindings u32[count,k] or None)."""
    values = np.zeros(count, np.float64)
    hits = np.zeros(count, np.uint8)
    binds = np.zeros((count, plan.k), np.uint32) if with_bindings else None
    _check(lib().agpm_ns_draw(dg._h, C.byref(plan), seed, first_id, count, _ptr(values, C.c_double),
                              _ptr(hits, C.c_uint8), None if binds is None else _ptr(binds, C.c_uint32), stream))
    return values, hits, binds


def run_fixed_budget(dg, plan, budget, seed, workers=1, stream=None):
    """run_fixed_budget (ns_engine.cpp:142-153); device streams are the
    reference's workers=1 streams whatever `workers` says."""
    acc = Accumulator()
    _check(lib().agpm_ns_fixed_budget(dg._h, C.byref(plan), budget, seed, C.byref(acc), stream))
    return acc


def hit_rate_report(dg, plan, sample_budget, seed, workers=1):
    acc = run_fixed_budget(dg, plan, sample_budget, seed, workers)
    return acc.hits / acc.n


def run_ns_online(dg, plan, eps, delta, policy=None, seed=1, workers=1, stream=None):
    """run_ns_online (ns_engine.cpp:106-140), workers=1 window semantics."""
    res = OnlineResult()
    pol = policy if policy is not None else OnlinePolicy()
    _check(lib().agpm_ns_online(dg._h, C.byref(plan), eps, delta, C.byref(pol), seed, C.byref(res), stream))
    return res


def exact_count(dg, plan, threads=1, stream=None):
    """exact_count (exact_engine.cpp:66-91) on the device; eager plans."""
    out = C.c_uint64()
    _check(lib().agpm_exact_count(dg._h, C.byref(plan), C.byref(out), stream))
    return out.value


def exact_count_shard(dg, plan, shard, nshards, stream=None):
    """One rank's share of exact_count: seeds of 32-arc chunks shard, shard + nshards, ...
    The shards sum to exact_count (all-reduce the partials across ranks)."""
    out = C.c_uint64()
    _check(lib().agpm_exact_count_shard(dg._h, C.byref(plan), shard, nshards, C.byref(out), stream))
    return out.value


def gs_estimate(dg, plan, scheme="color", keep_probability=1.0, colors=1, seed=0, threads=1, stream=None):
    """gs_estimate (gs_engine.cpp:42-75): scheme "color" (scale c^(k-1)) or "bernoulli" (scale p^-l)."""
    out = _abi.GsResult()
    _check(lib().agpm_gs_estimate(dg._h, C.byref(plan), {"bernoulli": 0, "color": 1}[scheme], keep_probability,
                                  colors, seed, C.byref(out), stream))
    return out


def gs_online(dg, plan, colors, eps, delta, max_colorings=4096, seed=1, stream=None):
    """Colour GS to eps at confidence 1 - delta: one colouring per coarse sample, NS online
    detector. OnlineResult: windows = colourings run."""
    out = _abi.OnlineResult()
    _check(lib().agpm_gs_online(dg._h, C.byref(plan), colors, eps, delta, max_colorings, seed, C.byref(out), stream))
    return out


def exact_count_rooted(dg, plan, root_limit, stream=None):
    out = C.c_uint64()
    _check(lib().agpm_exact_count_rooted(dg._h, C.byref(plan), root_limit, C.byref(out), stream))
    return out.value


REGION_METHODS = {"ns": 0, "gs": 1, "exact": 2}


def region_split(dg, plan, tau_degree, dense="ns", eps=0.01, delta=0.05, seed=1, colors=4, repeats=16,
                 max_samples=1000000000, stream=None):
    """Dense/sparse degree-threshold split (builder-defined):
    exact count of matches touching {deg < tau} + an estimate on the dense region."""
    out = _abi.RegionResult()
    _check(lib().agpm_region_split(dg._h, C.byref(plan), tau_degree, REGION_METHODS[dense], eps, delta, seed, colors,
                                   repeats, max_samples, C.byref(out), stream))
    return out


# ------------------------------------------------------------------ hybrid scheme choice
def choose_keep_probability(eps, delta, count_estimate, gamma_estimate):
    """choose_keep_probability (gs_engine.cpp:24-40) -> KeepProbability(p, sparsification_useless, color_count)."""
    out = _abi.KeepProbability()
    _check(lib().agpm_choose_keep_probability(eps, delta, count_estimate, gamma_estimate, C.byref(out)))
    return out


def ns_cost_cone(vertex_count, arc_count, plan, n_samples, hw_const):
    """ns_cost_cone (cost_model.cpp:92-110); average degree = arc_count / vertex_count."""
    out = _abi.CostCone()
    _check(lib().agpm_ns_cost_cone(vertex_count, arc_count, C.byref(plan), n_samples, hw_const, C.byref(out)))
    return out


def gs_cost_estimate(vertex_count, edge_count, plan, colors, hw_const, triangle_count):
    """gs_cost_estimate (cost_model.cpp:112-145)."""
    out = _abi.GsCost()
    _check(lib().agpm_gs_cost_estimate(vertex_count, edge_count, C.byref(plan), colors, hw_const, triangle_count,
                                       C.byref(out)))
    return out


def select_scheme(cone, gs):
    """select_scheme (cost_model.cpp:192-194): "gs" below the cone, else "ns"."""
    return "gs" if lib().agpm_select_scheme(C.byref(cone), C.byref(gs)) == 1 else "ns"


def count_matches_through_edge(graph, plan, u, v):
    out = C.c_uint64()
    _check(lib().agpm_count_matches_through_edge(graph._h, C.byref(plan), u, v, C.byref(out)))
    return out.value


def estimate_gamma(graph, plan, probe_edges, seed, work_budget=50000000):
    """estimate_gamma (gs_engine.cpp:179-197) on the host CSR."""
    out = C.c_uint64()
    _check(lib().agpm_estimate_gamma(graph._h, C.byref(plan), probe_edges, seed, work_budget, C.byref(out)))
    return out.value


def fast_profile(dg, plan, profile_fraction, user_epsilon, seed, profiler_sample_cap=1000000, stream=None):
    """fast_profile (cost_model.cpp:147-190): device Bernoulli sparsify + device online NS."""
    out = _abi.ProfileResult()
    _check(lib().agpm_fast_profile(dg._h, C.byref(plan), profile_fraction, user_epsilon, seed, profiler_sample_cap,
                                   C.byref(out), stream))
    return out


def calibrate_hardware_constant():
    out = C.c_double()
    _check(lib().agpm_calibrate_hardware_constant(C.byref(out)))
    return out.value


def count_hybrid(graph, dg, plan, eps, confidence, seed, profile_fraction=0.1, hw_const=1e-9, stream=None):
    """The CLI's loose mode (agpm_main.cpp:221-287): profile, gamma, keep probability, both cost
    models, select NS or GS, run it. Returns HybridResult (decision 0 = NS, 1 = GS)."""
    out = _abi.HybridResult()
    _check(lib().agpm_count_hybrid(graph._h, dg._h, C.byref(plan), eps, confidence, seed, profile_fraction, hw_const,
                                   C.byref(out), stream))
    return out


def bmin_bytes(dg, plan, seed, first_id, count, stream=None):
    out = C.c_uint64()
    _check(lib().agpm_ns_bmin_bytes(dg._h, C.byref(plan), seed, first_id, count, C.byref(out), stream))
    return out.value


def sample_dev(dg, plan, seed, first_id, count, d_values_ptr, stream=None):
    _check(lib().agpm_ns_sample_dev(dg._h, C.byref(plan), seed, first_id, count, C.c_void_p(d_values_ptr),
                                    None if stream is None else C.c_void_p(stream)))


def window_moments_dev(d_values_ptr, count, window, d_out_ptr, stream=None):
    _check(lib().agpm_window_moments_dev(C.c_void_p(d_values_ptr), count, window, C.c_void_p(d_out_ptr),
                                         None if stream is None else C.c_void_p(stream)))


STRATEGIES = {"auto": 0, "warp": 1, "lane": 2, "frontier": 3, "flat": 5}


def strategy_for(dg, plan, count):
    """Name of the sampler a launch of `count` ids would run under the current setting."""
    out = C.c_int(0)
    _check(lib().agpm_ns_strategy_for(dg._h, C.byref(plan), count, C.byref(out)))
    return {v: k for k, v in STRATEGIES.items()}[out.value]


def set_strategy(name):
    """Sampler kernel choice (all draw identical samples): auto | warp | lane | frontier | flat."""
    _check(lib().agpm_ns_set_strategy(STRATEGIES[name]))


def set_core_dim(dim):
    """Dense-core bit-matrix dimension (0 = off; None = auto: 65536 up to 2^21
    vertices, 262144 up to 2^25, 524288 above). Samples are identical for every setting."""
    _check(lib().agpm_ns_set_core_dim(0xFFFFFFFF if dim is None else int(dim)))


def set_rng(policy):
    """Per-sample stream: "counter" (CounterRng, the reference's stream; default) or "philox"
    (Philox4x32-10 keyed by the seed, counter (draw, sample id); flat sampler, eager plans)."""
    _check(lib().agpm_ns_set_rng({"counter": 0, "philox": 1}.get(policy, -1)))


def set_frontier_reuse(on):
    """Frontier sampler: reuse nested survivors between clique steps (same samples)."""
    _check(lib().agpm_ns_set_frontier_reuse(int(bool(on))))


# ------------------------------------------------------------------ multi-GPU
class Comm:
    """A rank communicator (agpm_comm): NCCL (one process per GPU) or a member
    of a LocalGroup (host threads of one process). Create it on the rank's GPU."""

    def __init__(self, handle, group=None):
        self._h = handle
        self._group = group  # keeps the group alive while a member exists

    @classmethod
    def nccl(cls, rank, world, unique_id):
        h = C.c_void_p()
        _check(lib().agpm_comm_init_nccl(rank, world, bytes(unique_id), C.byref(h)))
        return cls(h)

    def info(self):
        r, w, d, n = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        _check(lib().agpm_comm_info(self._h, C.byref(r), C.byref(w), C.byref(d), C.byref(n)))
        return {"rank": r.value, "world": w.value, "device": d.value, "nccl": bool(n.value)}

    def all_gather_dev(self, d_send_ptr, d_recv_ptr, bytes_per_rank, stream=None):
        """Enqueue recv[r * bytes ...] = rank r's send (device pointers) on `stream`."""
        _check(lib().agpm_comm_all_gather_dev(self._h, C.c_void_p(d_send_ptr), C.c_void_p(d_recv_ptr),
                                              bytes_per_rank, None if stream is None else C.c_void_p(stream)))

    def close(self):
        h = getattr(self, "_h", None)
        if h and h.value and _lib is not None:
            _lib.agpm_comm_free(h)
            self._h = None
        self._group = None

    def __del__(self):
        self.close()


class LocalGroup:
    """`world` ranks driven by host threads of this process (agpm_comm_group)."""

    def __init__(self, world):
        h = C.c_void_p()
        _check(lib().agpm_comm_group_create(world, C.byref(h)))
        self._h = h
        self.world = world

    def comm(self, rank):
        """The communicator of `rank`; call from the thread (and device) that drives it."""
        h = C.c_void_p()
        _check(lib().agpm_comm_init_local(self._h, rank, C.byref(h)))
        return Comm(h, self)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value and _lib is not None:
            _lib.agpm_comm_group_free(h)
            self._h = None


def nccl_unique_id():
    """ncclGetUniqueId (128 bytes): rank 0 makes it, the caller broadcasts it."""
    buf = C.create_string_buffer(_abi.NCCL_ID_BYTES)
    _check(lib().agpm_nccl_unique_id(buf))
    return buf.raw


def shard_round(launched, batch, window, max_samples, rank, world):
    """The id partition of one round of run_ns_online_sharded (host arithmetic)."""
    out = _abi.ShardRound()
    _check(lib().agpm_ns_shard_round(launched, batch, window, max_samples, rank, world, C.byref(out)))
    return out


def run_ns_online_sharded(comm, dg, plan, eps, delta, policy=None, seed=1, stream=None):
    """run_ns_online (ns_engine.cpp:106-140) over the ranks of `comm`: every rank
    passes its replica and gets the single-GPU (= reference workers=1) result."""
    res = OnlineResult()
    pol = policy if policy is not None else OnlinePolicy()
    _check(lib().agpm_ns_online_sharded(comm._h, dg._h, C.byref(plan), eps, delta, C.byref(pol), seed,
                                        C.byref(res), stream))
    return res


def run_fixed_budget_sharded(comm, dg, plan, budget, seed, stream=None):
    acc = Accumulator()
    _check(lib().agpm_ns_fixed_budget_sharded(comm._h, dg._h, C.byref(plan), budget, seed, C.byref(acc), stream))
    return acc


def exact_count_sharded(comm, dg, plan, stream=None):
    out = C.c_uint64()
    _check(lib().agpm_exact_count_sharded(comm._h, dg._h, C.byref(plan), C.byref(out), stream))
    return out.value


def kernel_launches():
    return lib().agpm_kernel_launches()


def sync(stream=None):
    """Wait for the library stream (or `stream`)."""
    _check(lib().agpm_sync(stream))


def device_count():
    n = C.c_int()
    _check(lib().agpm_device_count(C.byref(n)))
    return n.value
