"""TEST INFRASTRUCTURE: ctypes bindings to the two CPU checkers.

* Oracle  — oracle/liboracle.so, my plain-C restatement of the reference path
            (oracle/agpm_oracle.c). Always buildable (gcc, one file).
* RefLib  — oracle/_ref/libagpm_ref.so, the UNMODIFIED reference compiled from
            /root/reference/proj/src by oracle/Makefile, behind ref_shim.cpp.
            Built in this container; travels prebuilt to the GPU box.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import this.
"""
import ctypes as C
import os
import subprocess

import numpy as np

from paper_2405_03488_b200 import _abi
from paper_2405_03488_b200._abi import Accumulator, OnlinePolicy, OnlineResult, Plan, Report

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "liboracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libagpm_ref.so")
# the timing build of the same sources (-O3 -DNDEBUG -march=x86-64-v3, oracle/Makefile)
REF_FAST_SO = os.path.join(ORACLE_DIR, "_ref", "libagpm_ref_fast.so")
REF_FAST_FLAGS = "g++ -O3 -DNDEBUG -march=x86-64-v3 -fopenmp -std=c++20"
REF_FLAGS = "g++ -O3 -fopenmp -std=c++20 (the reference CMake Release flags)"


def cpu_has_x86_64_v3():
    try:
        with open("/proc/cpuinfo") as f:
            flags = next((ln for ln in f if ln.startswith("flags")), "").split()
        return all(x in flags for x in ("avx2", "bmi2", "fma", "movbe"))
    except OSError:
        return False


def timing_ref_so():
    """(path, flags) of the reference build bench.py times on this host."""
    if os.path.exists(REF_FAST_SO) and cpu_has_x86_64_v3():
        return REF_FAST_SO, REF_FAST_FLAGS
    return REF_SO, REF_FLAGS


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            return next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), "unknown")
    except OSError:
        return "unknown"

u32, u64, dbl, P = C.c_uint32, C.c_uint64, C.c_double, C.c_void_p
pu32, pu64, pdbl, pu8 = C.POINTER(u32), C.POINTER(u64), C.POINTER(dbl), C.POINTER(C.c_uint8)
pPlan, pAcc = C.POINTER(Plan), C.POINTER(Accumulator)


def _ptr(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def _b(s):
    return s.encode() if isinstance(s, str) else (s or b"")


def build_oracle(ref=True):
    """make -C oracle (restatement always; the reference only if its tree exists)."""
    target = "all" if ref else os.path.basename(ORACLE_SO)
    subprocess.run(["make", "-s", "-C", ORACLE_DIR, target if target == "all" else ORACLE_SO],
                   check=True, stdout=subprocess.DEVNULL)


class Oracle:
    """The plain-C restatement."""

    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            build_oracle(ref=False)
        L = C.CDLL(ORACLE_SO)
        graph = [u32, u64, pu64, pu64, pu32]
        sig = {
            "orc_rng_u64": (None, [u64, u64, u64, u64, pu64]),
            "orc_rng_below": (None, [u64, u64, u64, u64, u64, pu64]),
            "orc_rng_double": (None, [u64, u64, u64, u64, pdbl]),
            "orc_derive_key": (u64, [u64, u64, u64]),
            "orc_edge_keep": (C.c_int, [u64, u32, u32, dbl]),
            "orc_vertex_color": (u32, [u64, u32, u32]),
            "orc_norm_cdf": (dbl, [dbl]),
            "orc_inv_norm_cdf": (C.c_int, [dbl, pdbl]),
            "orc_predicted_error": (C.c_int, [pAcc, dbl, C.POINTER(Report)]),
            "orc_draw_records": (C.c_int, graph + [pPlan, u64, u64, u64, u64, pdbl, pu8, pu32]),
            "orc_fixed_budget": (C.c_int, graph + [pPlan, u64, u64, pAcc]),
            "orc_ns_online": (C.c_int, graph + [pPlan, dbl, dbl, C.POINTER(OnlinePolicy), u64,
                                                C.POINTER(OnlineResult)]),
            "orc_exact_count": (C.c_int, graph + [C.c_int, pPlan, pu64]),
            "orc_exact_count_shard": (C.c_int, graph + [C.c_int, pPlan, u32, u32, pu64]),
            "orc_draw_records_philox": (C.c_int, graph + [pPlan, u64, u64, u64, pdbl, pu8, pu32]),
            "orc_draw_records_mt": (C.c_int, graph + [pPlan, u64, u64, u64, pdbl, pu8, pu32, C.c_int]),
            "orc_ns_online_mt": (C.c_int, graph + [pPlan, dbl, dbl, C.POINTER(OnlinePolicy), u64,
                                                   C.POINTER(OnlineResult), C.c_int]),
            "orc_philox4x32_10": (None, [pu32, u32, u32]),
            "orc_gen_rmat_pairs": (None, [u32, u32, dbl, dbl, dbl, u64, pu32]),
            "orc_relabel_by_degree": (None, [u32, pu64, pu32, pu64, pu32]),
            "orc_write_binary_csr": (C.c_int, [C.c_char_p, u32, u64, pu64, pu32]),
            "orc_orient_by_degree": (None, [u32, pu64, pu32, pu64, pu32]),
            "orc_bernoulli_sparsify": (u64, [u32, pu64, pu32, dbl, u64, pu64, pu32]),
            "orc_triangle_count": (u64, [u32, pu64, pu32]),
            "orc_color_split": (u64, [u32, pu64, pu32, u32, u64, pu32, pu64, pu32]),
        }
        for k, (r, a) in sig.items():
            f = getattr(L, k)
            f.restype, f.argtypes = r, a
        self.L = L

    # rng
    def rng_u64(self, seed, s1, s2, count):
        out = np.zeros(count, np.uint64)
        self.L.orc_rng_u64(seed, s1, s2, count, _ptr(out, u64))
        return out

    def rng_below(self, seed, s1, s2, bound, count):
        out = np.zeros(count, np.uint64)
        self.L.orc_rng_below(seed, s1, s2, bound, count, _ptr(out, u64))
        return out

    def rng_double(self, seed, s1, s2, count):
        out = np.zeros(count, np.float64)
        self.L.orc_rng_double(seed, s1, s2, count, _ptr(out, dbl))
        return out

    def inv_norm_cdf(self, q):
        out = C.c_double()
        if self.L.orc_inv_norm_cdf(q, C.byref(out)) != 0:
            raise ValueError("quantile must be inside (0,1)")
        return out.value

    def predicted_error(self, acc, delta):
        rep = Report()
        if self.L.orc_predicted_error(C.byref(acc), delta, C.byref(rep)) != 0:
            raise ValueError("delta must be inside (0,1)")
        return rep

    @staticmethod
    def _g(off, nbr, end=None):
        off = np.ascontiguousarray(off, dtype=np.uint64)
        nbr = np.ascontiguousarray(nbr, dtype=np.uint32)
        n = len(off) - 1 if end is None else len(off)
        e = None if end is None else np.ascontiguousarray(end, dtype=np.uint64)
        return (off, nbr, e), (n, _ptr(off, u64), None if e is None else _ptr(e, u64), _ptr(nbr, u32))

    def draw_records(self, off, nbr, m, plan, seed, first, count, worker=0, end=None):
        keep, (n, po, pe, pn) = self._g(off, nbr, end)
        vals = np.zeros(count, np.float64)
        hits = np.zeros(count, np.uint8)
        binds = np.zeros((count, plan.k), np.uint32)
        st = self.L.orc_draw_records(n, m, po, pe, pn, C.byref(plan), seed, worker, first, count,
                                     _ptr(vals, dbl), _ptr(hits, C.c_uint8), _ptr(binds, u32))
        assert st == 0
        return vals, hits, binds

    def draw_records_mt(self, off, nbr, m, plan, seed, first, count, end=None, threads=None):
        """draw_records over all host cores (same records: one stream per sample id)."""
        keep, (n, po, pe, pn) = self._g(off, nbr, end)
        vals = np.zeros(count, np.float64)
        hits = np.zeros(count, np.uint8)
        binds = np.zeros((count, plan.k), np.uint32)
        st = self.L.orc_draw_records_mt(n, m, po, pe, pn, C.byref(plan), seed, first, count, _ptr(vals, dbl),
                                        _ptr(hits, C.c_uint8), _ptr(binds, u32), threads or os.cpu_count() or 1)
        assert st == 0
        return vals, hits, binds

    def ns_online_mt(self, off, nbr, m, plan, eps, delta, policy, seed, end=None, threads=None):
        """ns_online with the samples drawn on all host cores; accumulation and stop
        test sequential in id order, so the result is ns_online's bit for bit."""
        keep, (n, po, pe, pn) = self._g(off, nbr, end)
        res = OnlineResult()
        assert self.L.orc_ns_online_mt(n, m, po, pe, pn, C.byref(plan), eps, delta, C.byref(policy), seed,
                                       C.byref(res), threads or os.cpu_count() or 1) == 0
        return res

    def draw_records_philox(self, off, nbr, m, plan, seed, first, count, end=None):
        keep, (n, po, pe, pn) = self._g(off, nbr, end)
        vals = np.zeros(count, np.float64)
        hits = np.zeros(count, np.uint8)
        binds = np.zeros((count, plan.k), np.uint32)
        st = self.L.orc_draw_records_philox(n, m, po, pe, pn, C.byref(plan), seed, first, count,
                                            _ptr(vals, dbl), _ptr(hits, C.c_uint8), _ptr(binds, u32))
        assert st == 0
        return vals, hits, binds

    def philox4x32_10(self, ctr, key):
        c = np.array(ctr, np.uint32)
        self.L.orc_philox4x32_10(_ptr(c, u32), key[0], key[1])
        return [int(x) for x in c]

    def fixed_budget(self, off, nbr, m, plan, budget, seed):
        keep, (n, po, pe, pn) = self._g(off, nbr)
        acc = Accumulator()
        assert self.L.orc_fixed_budget(n, m, po, pe, pn, C.byref(plan), budget, seed, C.byref(acc)) == 0
        return acc

    def ns_online(self, off, nbr, m, plan, eps, delta, policy, seed):
        keep, (n, po, pe, pn) = self._g(off, nbr)
        res = OnlineResult()
        assert self.L.orc_ns_online(n, m, po, pe, pn, C.byref(plan), eps, delta, C.byref(policy), seed,
                                    C.byref(res)) == 0
        return res

    def exact_count(self, off, nbr, m, plan, oriented=False, end=None):
        keep, (n, po, pe, pn) = self._g(off, nbr, end)
        out = C.c_uint64()
        st = self.L.orc_exact_count(n, m, po, pe, pn, int(oriented), C.byref(plan), C.byref(out))
        if st != 0:
            raise ValueError("invalid exact_count arguments")
        return out.value

    def exact_count_shard(self, off, nbr, m, plan, shard, nshards, oriented=False, end=None):
        keep, (n, po, pe, pn) = self._g(off, nbr, end)
        out = C.c_uint64()
        st = self.L.orc_exact_count_shard(n, m, po, pe, pn, int(oriented), C.byref(plan), shard, nshards,
                                          C.byref(out))
        if st != 0:
            raise ValueError("invalid exact_count arguments")
        return out.value

    def color_split(self, off, nbr, c, seed):
        off = np.ascontiguousarray(off, dtype=np.uint64)
        nbr = np.ascontiguousarray(nbr, dtype=np.uint32)
        n = len(off) - 1
        colors = np.zeros(n, np.uint32)
        split = np.zeros(n, np.uint64)
        out = np.zeros(len(nbr), np.uint32)
        same = self.L.orc_color_split(n, _ptr(off, u64), _ptr(nbr, u32), c, seed, _ptr(colors, u32),
                                      _ptr(split, u64), _ptr(out, u32))
        return colors, split, out, same

    def rmat_pairs(self, scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1):
        """The benchmark RMAT edge list ((ef << scale), 2) u32 — the product generator restated."""
        pairs = np.empty(((edge_factor << scale), 2), np.uint32)
        self.L.orc_gen_rmat_pairs(scale, edge_factor, a, b, c, seed, _ptr(pairs, u32))
        return pairs

    def relabel_by_degree(self, off, nbr):
        off = np.ascontiguousarray(off, dtype=np.uint64)
        nbr = np.ascontiguousarray(nbr, dtype=np.uint32)
        n = len(off) - 1
        o_off = np.zeros(n + 1, np.uint64)
        o_nbr = np.zeros(max(len(nbr), 1), np.uint32)
        self.L.orc_relabel_by_degree(n, _ptr(off, u64), _ptr(nbr, u32), _ptr(o_off, u64), _ptr(o_nbr, u32))
        return o_off, o_nbr[: len(nbr)]

    def write_binary_csr(self, path, off, nbr, m):
        off = np.ascontiguousarray(off, dtype=np.uint64)
        nbr = np.ascontiguousarray(nbr, dtype=np.uint32)
        if self.L.orc_write_binary_csr(_b(path), len(off) - 1, m, _ptr(off, u64), _ptr(nbr, u32)) != 0:
            raise OSError(f"cannot write {path}")

    def triangle_count(self, off, nbr):
        off = np.ascontiguousarray(off, dtype=np.uint64)
        nbr = np.ascontiguousarray(nbr, dtype=np.uint32)
        return self.L.orc_triangle_count(len(off) - 1, _ptr(off, u64), _ptr(nbr, u32))

    def orient_by_degree(self, off, nbr):
        off = np.ascontiguousarray(off, dtype=np.uint64)
        nbr = np.ascontiguousarray(nbr, dtype=np.uint32)
        n = len(off) - 1
        o_off = np.zeros(n + 1, np.uint64)
        o_nbr = np.zeros(len(nbr) // 2 + 1, np.uint32)
        self.L.orc_orient_by_degree(n, _ptr(off, u64), _ptr(nbr, u32), _ptr(o_off, u64), _ptr(o_nbr, u32))
        return o_off, o_nbr[: int(o_off[-1])]

    def bernoulli_sparsify(self, off, nbr, p, seed):
        off = np.ascontiguousarray(off, dtype=np.uint64)
        nbr = np.ascontiguousarray(nbr, dtype=np.uint32)
        n = len(off) - 1
        o_off = np.zeros(n + 1, np.uint64)
        o_nbr = np.zeros(max(1, len(nbr)), np.uint32)
        kept = self.L.orc_bernoulli_sparsify(n, _ptr(off, u64), _ptr(nbr, u32), p, seed, _ptr(o_off, u64),
                                             _ptr(o_nbr, u32))
        return o_off, o_nbr[:kept]


class RefGraph:
    def __init__(self, ref, h):
        self.ref, self.h = ref, h

    def __del__(self):
        if self.h:
            self.ref.L.ref_graph_free(self.h)

    def info(self):
        n, m, arcs, o = u32(), u64(), u64(), C.c_int()
        self.ref.L.ref_graph_info(self.h, C.byref(n), C.byref(m), C.byref(arcs), C.byref(o))
        return n.value, m.value, arcs.value, bool(o.value)

    def arrays(self):
        n, m, arcs, _ = self.info()
        off = np.zeros(n + 1, np.uint64)
        nbr = np.zeros(max(arcs, 1), np.uint32)
        self.ref.L.ref_graph_arrays(self.h, _ptr(off, u64), _ptr(nbr, u32))
        return off, nbr[:arcs]


class RefLib:
    """The compiled, unmodified reference behind oracle/ref_shim.cpp."""

    available = os.path.exists(REF_SO)

    def __init__(self, path=None):
        path = path or REF_SO
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        ph = C.POINTER(P)
        s = C.c_char_p
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_rng_u64": (None, [u64, u64, u64, u64, pu64]),
            "ref_rng_below": (None, [u64, u64, u64, u64, u64, pu64]),
            "ref_rng_double": (None, [u64, u64, u64, u64, pdbl]),
            "ref_derive_key": (u64, [u64, u64, u64]),
            "ref_edge_keep": (C.c_int, [u64, u32, u32, dbl]),
            "ref_vertex_color": (u32, [u64, u32, u32]),
            "ref_norm_cdf": (dbl, [dbl]),
            "ref_inv_norm_cdf": (C.c_int, [dbl, pdbl]),
            "ref_predicted_error": (C.c_int, [pAcc, dbl, C.POINTER(Report)]),
            "ref_plan_compile": (C.c_int, [s, s, C.c_int, C.c_int, pPlan]),
            "ref_plan_scaling_rule": (C.c_int, [s, s, C.c_int, C.c_int, C.c_char_p, C.c_size_t]),
            "ref_automorphism_count": (C.c_int, [s, s, pu64]),
            "ref_builtin_names": (C.c_int, [C.c_char_p, C.c_size_t]),
            "ref_graph_free": (None, [P]),
            "ref_graph_from_edges": (C.c_int, [pu32, u64, u32, ph]),
            "ref_graph_from_csr": (C.c_int, [u32, u64, pu64, pu32, C.c_int, ph]),
            "ref_graph_er": (C.c_int, [u32, dbl, u64, ph]),
            "ref_graph_complete": (C.c_int, [u32, ph]),
            "ref_graph_cycle": (C.c_int, [u32, ph]),
            "ref_graph_path": (C.c_int, [u32, ph]),
            "ref_graph_star": (C.c_int, [u32, ph]),
            "ref_graph_load": (C.c_int, [s, ph]),
            "ref_graph_write_binary": (C.c_int, [P, s]),
            "ref_graph_orient": (C.c_int, [P, ph]),
            "ref_graph_bernoulli": (C.c_int, [P, dbl, u64, ph]),
            "ref_graph_info": (None, [P, C.POINTER(u32), pu64, pu64, C.POINTER(C.c_int)]),
            "ref_graph_arrays": (None, [P, pu64, pu32]),
            "ref_triangle_count": (u64, [P]),
            "ref_color_split": (C.c_int, [P, u32, u64, pu32, pu64, pu32, pu64]),
            "ref_merge_colors": (C.c_int, [P, u32, u64, pu32, u32, pu32, pu64, pu32, pu64]),
            "ref_draw_records": (C.c_int, [P, s, s, C.c_int, C.c_int, u64, u64, u64, u64, pdbl, pu8, pu32]),
            "ref_fixed_budget": (C.c_int, [P, s, s, C.c_int, C.c_int, u64, u64, C.c_int, pAcc]),
            "ref_ns_online": (C.c_int, [P, s, s, C.c_int, C.c_int, dbl, dbl, C.POINTER(OnlinePolicy), u64,
                                        C.c_int, C.POINTER(OnlineResult)]),
            "ref_exact_count": (C.c_int, [P, s, s, C.c_int, C.c_int, pu64, pu64]),
            "ref_exact_count_colored": (C.c_int, [P, s, s, u32, u64, C.c_int, pu64]),
            "ref_brute_force": (C.c_int, [P, s, s, pu64]),
            "ref_gs_estimate": (C.c_int, [P, s, s, C.c_int, dbl, u32, u64, C.c_int, pdbl, pu64, pdbl]),
            "ref_choose_keep_probability": (C.c_int, [dbl, dbl, dbl, dbl, pdbl, C.POINTER(C.c_int),
                                                      C.POINTER(u32)]),
            "ref_estimate_gamma": (C.c_int, [P, s, u64, u64, C.c_int64, pu64]),
            "ref_count_through_edge": (C.c_int, [P, s, u32, u32, pu64]),
            "ref_ns_cost_cone": (C.c_int, [P, s, u64, dbl, pdbl]),
            "ref_gs_cost_estimate": (C.c_int, [P, s, u32, dbl, u64, pdbl]),
            "ref_fast_profile": (C.c_int, [P, s, dbl, dbl, u64, C.c_int, u64, pdbl]),
        }
        for k, (r, a) in sig.items():
            f = getattr(L, k)
            f.restype, f.argtypes = r, a
        self.L = L

    def _chk(self, st):
        if st != 0:
            raise RuntimeError(f"reference error {st}: {self.L.ref_last_error().decode()}")

    def _mk(self, fn, *args):
        h = P()
        self._chk(fn(*args, C.byref(h)))
        return RefGraph(self, h)

    # graphs
    def er_graph(self, n, p, seed):
        return self._mk(self.L.ref_graph_er, n, p, seed)

    def complete(self, n):
        return self._mk(self.L.ref_graph_complete, n)

    def cycle(self, n):
        return self._mk(self.L.ref_graph_cycle, n)

    def path(self, n):
        return self._mk(self.L.ref_graph_path, n)

    def star(self, leaves):
        return self._mk(self.L.ref_graph_star, leaves)

    def from_edges(self, edges, min_n=0):
        e = np.ascontiguousarray(np.asarray(edges, dtype=np.uint32).reshape(-1, 2))
        return self._mk(self.L.ref_graph_from_edges, _ptr(e, u32), e.shape[0], min_n)

    def from_csr(self, off, nbr, m, oriented=False):
        off = np.ascontiguousarray(off, dtype=np.uint64)
        nbr = np.ascontiguousarray(nbr, dtype=np.uint32)
        return self._mk(self.L.ref_graph_from_csr, len(off) - 1, m, _ptr(off, u64), _ptr(nbr, u32), int(oriented))

    def load(self, path):
        return self._mk(self.L.ref_graph_load, _b(path))

    def orient(self, g):
        return self._mk(self.L.ref_graph_orient, g.h)

    def bernoulli(self, g, p, seed):
        return self._mk(self.L.ref_graph_bernoulli, g.h, p, seed)

    # plans
    def plan(self, spec, mode=0, sym=True, induced=""):
        plan = Plan()
        self._chk(self.L.ref_plan_compile(_b(spec), _b(induced), mode, int(sym), C.byref(plan)))
        return plan

    def plan_error(self, spec, mode=0, sym=True, induced=""):
        plan = Plan()
        st = self.L.ref_plan_compile(_b(spec), _b(induced), mode, int(sym), C.byref(plan))
        return st, (self.L.ref_last_error().decode() if st else "")

    def scaling_rule(self, spec, mode=0, sym=True, induced=""):
        buf = C.create_string_buffer(512)
        self._chk(self.L.ref_plan_scaling_rule(_b(spec), _b(induced), mode, int(sym), buf, 512))
        return buf.value.decode()

    def automorphism_count(self, spec, induced=""):
        out = u64()
        self._chk(self.L.ref_automorphism_count(_b(spec), _b(induced), C.byref(out)))
        return out.value

    # engines
    def draw_records(self, g, spec, seed, first, count, mode=0, sym=True, induced="", worker=0):
        plan = self.plan(spec, mode, sym, induced)
        vals = np.zeros(count, np.float64)
        hits = np.zeros(count, np.uint8)
        binds = np.zeros((count, plan.k), np.uint32)
        self._chk(self.L.ref_draw_records(g.h, _b(spec), _b(induced), mode, int(sym), seed, worker, first, count,
                                          _ptr(vals, dbl), _ptr(hits, C.c_uint8), _ptr(binds, u32)))
        return vals, hits, binds

    def fixed_budget(self, g, spec, budget, seed, workers=1, mode=0, induced=""):
        acc = Accumulator()
        self._chk(self.L.ref_fixed_budget(g.h, _b(spec), _b(induced), mode, 1, budget, seed, workers, C.byref(acc)))
        return acc

    def ns_online(self, g, spec, eps, delta, policy, seed, workers=1, mode=0, induced=""):
        res = OnlineResult()
        self._chk(self.L.ref_ns_online(g.h, _b(spec), _b(induced), mode, 1, eps, delta, C.byref(policy), seed,
                                       workers, C.byref(res)))
        return res

    def exact_count(self, g, spec, threads=1, sym=True, induced=""):
        c, w = u64(), u64()
        self._chk(self.L.ref_exact_count(g.h, _b(spec), _b(induced), int(sym), threads, C.byref(c), C.byref(w)))
        return c.value

    def exact_count_colored(self, g, spec, colors, seed, threads=1, induced=""):
        c = u64()
        self._chk(self.L.ref_exact_count_colored(g.h, _b(spec), _b(induced), colors, seed, threads, C.byref(c)))
        return c.value

    def brute_force(self, g, spec, induced=""):
        c = u64()
        self._chk(self.L.ref_brute_force(g.h, _b(spec), _b(induced), C.byref(c)))
        return c.value

    def color_split(self, g, c, seed):
        n, m, arcs, _ = g.info()
        colors = np.zeros(n, np.uint32)
        split = np.zeros(n, np.uint64)
        nbr = np.zeros(max(arcs, 1), np.uint32)
        same = u64()
        self._chk(self.L.ref_color_split(g.h, c, seed, _ptr(colors, u32), _ptr(split, u64), _ptr(nbr, u32),
                                         C.byref(same)))
        return colors, split, nbr[:arcs], same.value

    def merge_colors(self, g, c, seed, group_map):
        n, m, arcs, _ = g.info()
        gm = np.asarray(group_map, np.uint32)
        colors = np.zeros(n, np.uint32)
        split = np.zeros(n, np.uint64)
        nbr = np.zeros(max(arcs, 1), np.uint32)
        same = u64()
        self._chk(self.L.ref_merge_colors(g.h, c, seed, _ptr(gm, u32), len(gm), _ptr(colors, u32), _ptr(split, u64),
                                          _ptr(nbr, u32), C.byref(same)))
        return colors, split, nbr[:arcs], same.value

    def gs_estimate(self, g, spec, scheme, p=1.0, colors=1, seed=0, threads=1, induced=""):
        est, raw, scale = dbl(), u64(), dbl()
        self._chk(self.L.ref_gs_estimate(g.h, _b(spec), _b(induced), scheme, p, colors, seed, threads,
                                         C.byref(est), C.byref(raw), C.byref(scale)))
        return est.value, raw.value, scale.value

    def triangle_count(self, g):
        return self.L.ref_triangle_count(g.h)


def reference_rmat_graph(scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1, path=None, ref_path=None):
    """The benchmark RMAT graph built WITHOUT the product library (bench.py's
    reference arm): edges from the oracle's generator restatement, CSR from the
    reference's own CsrGraph::from_edges (csr_graph.cpp:46-72), the oracle's
    (degree, id) relabel, written as AGPM v1 and read back through the
    reference's load_graph_auto (csr_graph.cpp:143-170). Returns (RefLib, RefGraph)."""
    import tempfile

    O, R = Oracle(), RefLib(ref_path)
    g0 = R.from_edges(O.rmat_pairs(scale, edge_factor, a, b, c, seed), 1 << scale)
    m = g0.info()[1]
    off, nbr = O.relabel_by_degree(*g0.arrays())
    del g0
    own = path is None
    if own:
        fd, path = tempfile.mkstemp(suffix=".agpm")
        os.close(fd)
    try:
        O.write_binary_csr(path, off, nbr, m)
        del off, nbr
        return R, R.load(path)
    finally:
        if own:
            os.unlink(path)
