"""ctypes binding of libgmt_b200.so (the C ABI in include/gmt_b200.h).

There is deliberately no fallback: if the shared library is missing this
module raises at import, and every compute call fails with NoDeviceError
when no B200 is present.  Build with ``python -m paper_1705_02403_b200.build``.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import abi
from .errors import raise_for
from .graph import Graph

LIB_PATH = os.environ.get("GMT_B200_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libgmt_b200.so")

_dp = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u8p = C.POINTER(C.c_uint8)
_P = C.POINTER
_vp = C.c_void_p

# (name, restype, argtypes) for every symbol the header declares.
SIGNATURES = [
    ("gmt_last_error", C.c_char_p, []),
    ("gmt_abi_version", C.c_int, []),
    ("gmt_struct_sizes", C.c_int, [_i64p, C.c_int32]),
    ("gmt_ctx_create", C.c_int, [C.c_int, _P(_vp)]),
    ("gmt_ctx_destroy", None, [_vp]),
    ("gmt_ctx_stream", _vp, [_vp]),
    ("gmt_ctx_synchronize", C.c_int, [_vp]),
    ("gmt_launch_count", C.c_int64, [_vp]),
    ("gmt_ctx_set_option", C.c_int, [_vp, C.c_int, C.c_int64]),
    ("gmt_ctx_counters", C.c_int, [_vp, _i64p, C.c_int32]),
    ("gmt_unit_ball_volume", C.c_int, [C.c_int32, _dp]),
    ("gmt_connection_radius", C.c_int, [C.c_int32, C.c_int64, C.c_double, C.c_double, _dp]),
    ("gmt_sample_free", C.c_int, [_vp, C.c_int32, _P(abi.Scene), _P(abi.SampleSource), _dp, _dp,
                                  _i32p, _i32p]),
    ("gmt_append_init", C.c_int, [_vp, C.c_int32, _dp, _dp, _i32p, _dp, C.c_int32, C.c_double,
                                  _dp, _dp, _i32p, _i32p, _i32p]),
    ("gmt_build_neighbor_graph", C.c_int, [_vp, _dp, C.c_int32, C.c_int32, C.c_double, _i64p,
                                           _i64p, _i32p, _dp]),
    ("gmt_di_costs", C.c_int, [_vp, _dp, _dp, C.c_int64, _P(abi.DiParams), _dp, _dp]),
    ("gmt_quad_costs", C.c_int, [_vp, _dp, _dp, C.c_int64, _P(abi.QuadParams), _dp, _dp]),
    ("gmt_build_quad_graph", C.c_int, [_vp, _dp, C.c_int32, _P(abi.QuadParams), C.c_double,
                                       _i64p, _i64p, _i32p, _dp, _dp, _i64p, _i32p, _dp, _i32p,
                                       _dp]),
    ("gmt_build_di_graph", C.c_int, [_vp, _dp, C.c_int32, _P(abi.DiParams), C.c_double, _i64p,
                                     _i64p, _i32p, _dp, _dp, _i64p, _i32p, _dp, _i32p, _dp]),
    ("gmt_problem_key", C.c_int, [_P(abi.Problem), _P(C.c_uint64)]),
    ("gmt_dubins_costs", C.c_int, [_vp, _dp, _dp, C.c_int64, C.c_int32, _P(abi.DubinsParams), _dp,
                                   _i32p]),
    ("gmt_plan_problems", C.c_int, [_vp, _P(abi.Problem), C.c_int32, _i32p, _P(abi.PlanSummary),
                                    C.c_int32, _dp]),
    ("gmt_run_trial", C.c_int, [_vp, _P(abi.Scenario), C.c_uint64, _P(abi.TrialOutcome), _dp,
                                C.c_int64]),
    ("gmt_run_campaign", C.c_int, [C.c_int, _P(abi.Scenario), _dp, C.c_int32, _dp, C.c_int32, _dp,
                                   C.c_int32, C.c_int32, _i32p]),
    ("gmt_graph_cache_save", C.c_int, [C.c_char_p, C.c_uint64, C.c_int32, C.c_double, _i64p, _i32p,
                                       _dp]),
    ("gmt_graph_cache_load", C.c_int, [C.c_char_p, C.c_uint64, C.c_int32, C.c_double, _i32p, _i64p, C.c_int64,
                                       _i64p, _i32p, _dp]),
    ("gmt_instance_build_cached", C.c_int, [_vp, _P(abi.Problem), C.c_char_p, _P(_vp), _i32p]),
    ("gmt_instance_cache_save", C.c_int, [_vp, _vp, C.c_char_p, C.c_uint64]),
    ("gmt_instance_upload", C.c_int, [_vp, _P(abi.Scene), _dp, C.c_int32, C.c_int32,
                                      _P(abi.GraphView), _P(_vp)]),
    ("gmt_instance_build", C.c_int, [_vp, _P(abi.Problem), _P(_vp)]),
    ("gmt_instance_info", C.c_int, [_vp, _i32p, _i32p, _i32p, _dp, _i64p, _i32p]),
    ("gmt_instance_download", C.c_int, [_vp, _vp, _dp, _i32p, _i64p, _i32p, _dp]),
    ("gmt_instance_destroy", None, [_vp]),
    ("gmt_plan", C.c_int, [_vp, _vp, C.c_int32, C.c_double, C.c_double, _P(abi.PlanOut)]),
    ("gmt_plan_host", C.c_int, [_vp, _P(abi.Scene), _dp, C.c_int32, C.c_int32, _P(abi.GraphView),
                                C.c_int32, C.c_double, C.c_double, _P(abi.PlanOut)]),
    ("gmt_fmt_plan", C.c_int, [_vp, _vp, C.c_int32, _P(abi.PlanOut)]),
    ("gmt_dijkstra_oracle", C.c_int, [_vp, _vp, C.c_int32, _P(abi.PlanOut)]),
    ("gmt_batch_create", C.c_int, [_vp, C.c_int32, _P(_vp), _i32p, C.c_double, _P(_vp)]),
    ("gmt_batch_create_problems", C.c_int, [_vp, _P(abi.Problem), C.c_int32, _i32p, _P(_vp)]),
    ("gmt_ctx_pool_info", C.c_int, [_vp, _i32p, _i64p, _dp, _i32p, _dp]),
    ("gmt_batch_graph", C.c_int, [_vp, _vp, C.c_int32, _i32p, _i64p, _i64p, _dp, _i64p, _i32p, _dp, _dp,
                                  _i64p, _i32p]),
    ("gmt_batch_launch", C.c_int, [_vp, _vp]),
    ("gmt_batch_summaries", C.c_int, [_vp, _vp, _P(abi.PlanSummary)]),
    ("gmt_batch_result", C.c_int, [_vp, _vp, C.c_int32, _P(abi.PlanOut)]),
    ("gmt_batch_destroy", None, [_vp]),
    ("gmt_plan_batch_host", C.c_int, [_vp, _P(abi.BatchHost), C.c_double, _P(abi.PlanSummary),
                                      _i32p, _u8p, _dp, _i32p, _i64p]),
    ("gmt_segment_free", C.c_int, [_vp, C.c_int32, C.c_int32, _dp, _dp, _dp, _dp, C.c_int64, _u8p]),
    ("gmt_problem_parse", C.c_int, [C.c_char_p, C.c_size_t, _P(_vp)]),
    ("gmt_problem_load", C.c_int, [C.c_char_p, _P(_vp)]),
    ("gmt_problem_file_view", C.c_int, [_vp, _P(abi.Problem), _P(C.c_char_p)]),
    ("gmt_problem_file_destroy", None, [_vp]),
    ("gmt_host_alloc", C.c_int, [C.c_size_t, _P(_vp)]),
    ("gmt_host_free", None, [_vp]),
]

OPT_CLUSTER = 1
OPT_THREADS = 2
OPT_BATCH_THREADS = 3
OPT_BATCH_CLUSTER = 4
OPT_COUNTERS = 5


def load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run `python -m paper_1705_02403_b200.build` "
                          "(the B200 library has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        if os.environ.get("GMT_B200_LIB") and not hasattr(lib, name):
            continue  # an older experimental build (A/B timing) may lack newer entry points
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib: C.CDLL | None = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        _lib = load()
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        raise_for(rc, lib().gmt_last_error().decode())


class ProblemBatch:
    """gmt_problem structs of many ProblemSpecs, flattened once (the specs
    keep the arrays the structs point to alive)."""

    def __init__(self, specs):
        self.specs = list(specs)
        self.count = len(self.specs)
        self.dim = self.specs[0].dim
        self.array = (abi.Problem * self.count)()
        self._keep = []
        for q, sp in enumerate(self.specs):
            self.array[q] = sp.flat()
            self._keep.append(sp._keep)  # the arrays this struct points to


class Instance:
    """A device-resident ProblemInstance (problem.hpp:52-57)."""

    def __init__(self, ctx: "Context", handle: C.c_void_p, spec=None):
        self.ctx = ctx
        self.h = handle
        self.spec = spec
        n, d, ii, gc = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        r = C.c_double()
        ne = C.c_int64()
        check(lib().gmt_instance_info(self.h, C.byref(n), C.byref(d), C.byref(ii), C.byref(r),
                                      C.byref(ne), C.byref(gc)))
        self.n, self.dim, self.init_index = n.value, d.value, ii.value
        self.radius, self.num_edges, self.goal_count = r.value, ne.value, gc.value

    def cache_save(self, file: str, key: int) -> None:
        """save_graph_cache (graph.cpp:240-276) of this instance's graph."""
        check(lib().gmt_instance_cache_save(self.ctx.h, self.h, os.fsencode(file), key))

    def download(self, goal: bool = True):
        """-> (coords [n, dim], goal_idx, Graph)"""
        coords = np.zeros(self.n * self.dim)
        gidx = np.zeros(max(self.goal_count, 1), np.int32)
        ptr = np.zeros(self.n + 1, np.int64)
        col = np.zeros(max(self.num_edges, 1), np.int32)
        cost = np.zeros(max(self.num_edges, 1))
        check(lib().gmt_instance_download(
            self.ctx.h, self.h, abi.ptr(coords, C.c_double),
            abi.ptr(gidx if goal else None, C.c_int32), abi.ptr(ptr, C.c_int64),
            abi.ptr(col, C.c_int32), abi.ptr(cost, C.c_double)))
        g = Graph(self.n, self.radius, ptr, col[: self.num_edges], cost[: self.num_edges],
                  dim=self.dim)
        return coords.reshape(self.n, self.dim), gidx[: self.goal_count], g

    def close(self):
        if self.h:
            lib().gmt_instance_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Batch:
    """gmt_batch.  Its solve jobs point into the instances' device memory, so
    the Batch holds a reference to every Instance for its own lifetime."""

    def __init__(self, ctx: "Context", handle, count: int, sizes, instances=()):
        self.ctx, self.h, self.count, self.sizes = ctx, handle, count, sizes
        self._insts = list(instances)

    def launch(self):
        check(lib().gmt_batch_launch(self.ctx.h, self.h))

    def summaries(self):
        out = (abi.PlanSummary * self.count)()
        check(lib().gmt_batch_summaries(self.ctx.h, self.h, out))
        return list(out)

    def graph(self, q: int) -> dict:
        """Query q's graph (gmt_batch_graph): coords, in-rows with costs and
        durations, out-row targets, as host arrays."""
        n, ni, no = C.c_int32(), C.c_int64(), C.c_int64()
        z = lambda t: abi.ptr(None, t)  # noqa: E731
        check(lib().gmt_batch_graph(self.ctx.h, self.h, q, C.byref(n), C.byref(ni), C.byref(no), z(C.c_double),
                                    z(C.c_int64), z(C.c_int32), z(C.c_double), z(C.c_double), z(C.c_int64),
                                    z(C.c_int32)))
        V = n.value
        g = dict(n=V, in_ptr=np.zeros(V + 1, np.int64), in_col=np.zeros(max(ni.value, 1), np.int32),
                 in_cost=np.zeros(max(ni.value, 1)), in_tau=np.zeros(max(ni.value, 1)),
                 out_ptr=np.zeros(V + 1, np.int64), out_col=np.zeros(max(no.value, 1), np.int32))
        coords = np.zeros(V * 16)
        check(lib().gmt_batch_graph(self.ctx.h, self.h, q, C.byref(n), C.byref(ni), C.byref(no),
                                    abi.ptr(coords, C.c_double), abi.ptr(g["in_ptr"], C.c_int64),
                                    abi.ptr(g["in_col"], C.c_int32), abi.ptr(g["in_cost"], C.c_double),
                                    abi.ptr(g["in_tau"], C.c_double), abi.ptr(g["out_ptr"], C.c_int64),
                                    abi.ptr(g["out_col"], C.c_int32)))
        for k, m in (("in_col", ni.value), ("in_cost", ni.value), ("in_tau", ni.value), ("out_col", no.value)):
            g[k] = g[k][:m]
        g["coords"] = coords
        return g

    def result(self, q: int) -> abi.PlanResultPy:
        if self.sizes[q] is None:
            self.sizes[q] = self.graph(q)["n"]
        buf = abi.PlanBuffers(self.sizes[q])
        check(lib().gmt_batch_result(self.ctx.h, self.h, q, C.byref(buf.out)))
        return buf.result()

    def close(self):
        if self.h:
            lib().gmt_batch_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Context:
    """gmt_ctx: one device, one stream."""

    def __init__(self, device: int = 0):
        self.h = C.c_void_p()
        check(lib().gmt_ctx_create(device, C.byref(self.h)))
        self.device = device

    @property
    def stream(self) -> int:
        return lib().gmt_ctx_stream(self.h) or 0

    @property
    def launch_count(self) -> int:
        return lib().gmt_launch_count(self.h)

    def set_option(self, opt: int, value: int):
        check(lib().gmt_ctx_set_option(self.h, opt, value))

    def synchronize(self):
        check(lib().gmt_ctx_synchronize(self.h))

    def counters(self, reset: bool = False) -> dict:
        """Traffic counts of the solves launched while OPT_COUNTERS was on."""
        out = np.zeros(3, np.int64)
        check(lib().gmt_ctx_counters(self.h, abi.ptr(out, C.c_int64), 1 if reset else 0))
        return {"in_scan": int(out[0]), "out_scan": int(out[1]), "open_parent_reads": int(out[2])}

    def close(self):
        if self.h:
            lib().gmt_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- offline phase ---------------------------------------------------
    @staticmethod
    def connection_radius(dim: int, n: int, eta: float = 0.0, mu: float = 1.0) -> float:
        out = C.c_double()
        check(lib().gmt_connection_radius(dim, n, eta, mu, C.byref(out)))
        return out.value

    @staticmethod
    def unit_ball_volume(d: int) -> float:
        out = C.c_double()
        check(lib().gmt_unit_ball_volume(d, C.byref(out)))
        return out.value

    def sample_free(self, spec, n: int | None = None):
        n = spec.n if n is None else n
        coords = np.zeros(n * spec.dim)
        gidx = np.zeros(n + 1, np.int32)
        gc = C.c_int32()
        sc, src = spec.scene(), spec.source()
        check(lib().gmt_sample_free(self.h, n, C.byref(sc), C.byref(src), abi.ptr(coords, C.c_double),
                                    abi.ptr(None, C.c_double), abi.ptr(gidx, C.c_int32),
                                    C.byref(gc)))
        return coords.reshape(n, spec.dim), gidx[: gc.value].copy()

    def append_init(self, coords, goal_idx, init, goal_lo, goal_hi):
        n0, dim = coords.shape
        buf = np.zeros((n0 + 1) * dim)
        buf[: n0 * dim] = coords.reshape(-1)
        g = np.zeros(n0 + 2, np.int32)
        g[: len(goal_idx)] = goal_idx
        n = C.c_int32(n0)
        gc = C.c_int32(len(goal_idx))
        idx = C.c_int32()
        init, gl, gh = abi.f64(init), abi.f64(goal_lo), abi.f64(goal_hi)
        check(lib().gmt_append_init(self.h, dim, abi.ptr(buf, C.c_double), abi.ptr(None, C.c_double),
                                    C.byref(n), abi.ptr(init, C.c_double), 0, 0.0,
                                    abi.ptr(gl, C.c_double), abi.ptr(gh, C.c_double),
                                    abi.ptr(g, C.c_int32), C.byref(gc), C.byref(idx)))
        return buf[: n.value * dim].reshape(n.value, dim), g[: gc.value].copy(), idx.value

    def segment_free(self, spec, a, b) -> np.ndarray:
        """segment_free (space.cpp:80-90) of rows a[i] -> b[i] against
        spec's boxes, on the device (the lazy check's own warp test)."""
        a = abi.f64(a).reshape(-1, spec.dim)
        b = abi.f64(b).reshape(-1, spec.dim)
        if a.shape != b.shape:
            raise ValueError("a and b differ in shape")
        lo, hi = abi.f64(spec.box_lo).reshape(-1), abi.f64(spec.box_hi).reshape(-1)
        out = np.zeros(a.shape[0], np.uint8)
        check(lib().gmt_segment_free(self.h, spec.dim, spec.num_boxes, abi.ptr(lo, C.c_double),
                                     abi.ptr(hi, C.c_double), abi.ptr(a, C.c_double),
                                     abi.ptr(b, C.c_double), a.shape[0], abi.ptr(out, C.c_uint8)))
        return out.astype(bool)

    def build_neighbor_graph(self, coords, radius: float) -> Graph:
        coords = abi.f64(coords)
        n, dim = coords.shape
        ne = C.c_int64()
        check(lib().gmt_build_neighbor_graph(self.h, abi.ptr(coords, C.c_double), n, dim, radius,
                                             C.byref(ne), abi.ptr(None, C.c_int64),
                                             abi.ptr(None, C.c_int32), abi.ptr(None, C.c_double)))
        ptr = np.zeros(n + 1, np.int64)
        col = np.zeros(max(ne.value, 1), np.int32)
        cost = np.zeros(max(ne.value, 1))
        check(lib().gmt_build_neighbor_graph(self.h, abi.ptr(coords, C.c_double), n, dim, radius,
                                             C.byref(ne), abi.ptr(ptr, C.c_int64),
                                             abi.ptr(col, C.c_int32), abi.ptr(cost, C.c_double)))
        return Graph(n, radius, ptr, col[: ne.value], cost[: ne.value], dim=dim)

    # ---- double integrator (NEW model) ----------------------
    def di_costs(self, x0s, x1s, params: abi.DiParams):
        """Device cost and duration of each state pair (rows of x0s, x1s)."""
        return self._kino_costs(lib().gmt_di_costs, 6, x0s, x1s, params)

    def build_di_graph(self, coords, params: abi.DiParams, radius: float,
                       paths: bool = True) -> Graph:
        """Directed DI graph (out-rows, in-rows, optional waypoint paths) as a
        reference-shaped Graph: path ids = out-edge indices."""
        return self._kino_graph(lib().gmt_build_di_graph, 6, coords, params, radius, paths)

    # ---- Dubins airplane (steering.cpp:53-112) ------------------------------
    def dubins_costs(self, x0s, x1s, dim: int, params: abi.DubinsParams):
        """connect_cost and segment counts of (x, y[, z], heading) state pairs."""
        x0s = abi.f64(x0s).reshape(-1, dim + 1)
        x1s = abi.f64(x1s).reshape(-1, dim + 1)
        m = x0s.shape[0]
        cost, segs = np.zeros(m), np.zeros(m, np.int32)
        check(lib().gmt_dubins_costs(self.h, abi.ptr(x0s, C.c_double), abi.ptr(x1s, C.c_double), m, dim,
                                     C.byref(params), abi.ptr(cost, C.c_double), abi.ptr(segs, C.c_int32)))
        return cost, segs

    # ---- quadrotor (NEW model) ------------------------------
    def quad_costs(self, x0s, x1s, params: abi.QuadParams):
        return self._kino_costs(lib().gmt_quad_costs, 12, x0s, x1s, params)

    def build_quad_graph(self, coords, params: abi.QuadParams, radius: float,
                         paths: bool = True) -> Graph:
        return self._kino_graph(lib().gmt_build_quad_graph, 12, coords, params, radius, paths)

    def _kino_costs(self, fn, dim, x0s, x1s, params):
        x0s, x1s = abi.f64(x0s).reshape(-1, dim), abi.f64(x1s).reshape(-1, dim)
        m = x0s.shape[0]
        cost, tau = np.zeros(m), np.zeros(m)
        check(fn(self.h, abi.ptr(x0s, C.c_double), abi.ptr(x1s, C.c_double), m, C.byref(params),
                 abi.ptr(cost, C.c_double), abi.ptr(tau, C.c_double)))
        return cost, tau

    def _kino_graph(self, fn, dim, coords, params, radius, paths) -> Graph:
        coords = abi.f64(coords)
        n = coords.shape[0]
        ne = C.c_int64()
        z = lambda t: abi.ptr(None, t)  # noqa: E731
        check(fn(self.h, abi.ptr(coords, C.c_double), n, C.byref(params), radius, C.byref(ne),
                 z(C.c_int64), z(C.c_int32), z(C.c_double), z(C.c_double), z(C.c_int64),
                 z(C.c_int32), z(C.c_double), z(C.c_int32), z(C.c_double)))
        E = ne.value
        M1 = params.segments + 1
        optr, iptr = np.zeros(n + 1, np.int64), np.zeros(n + 1, np.int64)
        ocol, icol = np.zeros(max(E, 1), np.int32), np.zeros(max(E, 1), np.int32)
        ocost, icost, otau = np.zeros(max(E, 1)), np.zeros(max(E, 1)), np.zeros(max(E, 1))
        ipath = np.zeros(max(E, 1), np.int32) if paths else None
        pts = np.zeros(max(E, 1) * M1 * dim) if paths else None
        check(fn(self.h, abi.ptr(coords, C.c_double), n, C.byref(params), radius, C.byref(ne),
                 abi.ptr(optr, C.c_int64), abi.ptr(ocol, C.c_int32), abi.ptr(ocost, C.c_double),
                 abi.ptr(otau, C.c_double), abi.ptr(iptr, C.c_int64), abi.ptr(icol, C.c_int32),
                 abi.ptr(icost, C.c_double), abi.ptr(ipath, C.c_int32), abi.ptr(pts, C.c_double)))
        g = Graph(n, radius, optr, ocol[:E], ocost[:E], dim=dim, directed=True, in_ptr=iptr,
                  in_col=icol[:E], in_cost=icost[:E],
                  out_path=np.arange(E, dtype=np.int32) if paths else None,
                  in_path=None if ipath is None else ipath[:E],
                  path_ptr=np.arange(E + 1, dtype=np.int64) * M1 if paths else None,
                  path_pts=None if pts is None else pts[: E * M1 * dim])
        g.out_tau = otau[:E]
        return g

    def build_instance(self, spec) -> Instance:
        h = C.c_void_p()
        p = spec.flat()
        check(lib().gmt_instance_build(self.h, C.byref(p), C.byref(h)))
        return Instance(self, h, spec)

    def build_instance_cached(self, spec, cache_file: str):
        """build_instance(p, workers, cache_file) (problem.cpp:336-363) ->
        (Instance, cache_hit)."""
        h = C.c_void_p()
        hit = C.c_int32()
        p = spec.flat()
        check(lib().gmt_instance_build_cached(self.h, C.byref(p), os.fsencode(cache_file), C.byref(h),
                                              C.byref(hit)))
        return Instance(self, h, spec), bool(hit.value)

    def upload(self, spec, coords, goal_count: int, graph: Graph) -> Instance:
        coords = abi.f64(coords)
        h = C.c_void_p()
        sc = spec.scene()
        gv = graph.view()
        check(lib().gmt_instance_upload(self.h, C.byref(sc), abi.ptr(coords, C.c_double),
                                        coords.shape[0], goal_count, C.byref(gv), C.byref(h)))
        return Instance(self, h, spec)

    # ---- online phase ----------------------------------------------------
    def plan(self, inst: Instance, init_index: int | None = None, lam: float = 1.0,
             radius: float | None = None) -> abi.PlanResultPy:
        buf = abi.PlanBuffers(inst.n)
        ii = inst.init_index if init_index is None else init_index
        r = inst.radius if radius is None else radius
        check(lib().gmt_plan(self.h, inst.h, ii, lam, r, C.byref(buf.out)))
        return buf.result()

    def fmt_plan(self, inst: Instance, init_index: int | None = None) -> abi.PlanResultPy:
        buf = abi.PlanBuffers(inst.n)
        ii = inst.init_index if init_index is None else init_index
        check(lib().gmt_fmt_plan(self.h, inst.h, ii, C.byref(buf.out)))
        return buf.result()

    def dijkstra_oracle(self, inst: Instance, init_index: int | None = None) -> abi.PlanResultPy:
        """dijkstra_oracle (planner.cpp:264-334) on the device: eager checks
        of every edge, then exact Dijkstra."""
        buf = abi.PlanBuffers(inst.n)
        ii = inst.init_index if init_index is None else init_index
        check(lib().gmt_dijkstra_oracle(self.h, inst.h, ii, C.byref(buf.out)))
        return buf.result()

    def plan_problems(self, specs, path_cap: int = 0):
        """build_instance + gmt_plan for a batch of Euclidean problems, or of
        double-integrator problems over the shared sample pool (one batched
        offline phase, one batched solve).  `specs`: ProblemSpecs or
        a ProblemBatch (flattened once, reusable).  -> (status codes,
        summaries, path states [count, path_cap, dim] or None)."""
        pb = specs if isinstance(specs, ProblemBatch) else ProblemBatch(specs)
        count = pb.count
        probs = pb.array
        status = np.zeros(count, np.int32)
        summ = (abi.PlanSummary * count)()
        d = pb.dim
        paths = np.zeros(max(count * path_cap * d, 1)) if path_cap > 0 else None
        check(lib().gmt_plan_problems(self.h, probs, count, abi.ptr(status, C.c_int32), summ, path_cap,
                                      abi.ptr(paths, C.c_double)))
        return status, list(summ), (paths[: count * path_cap * d].reshape(count, path_cap, d)
                                    if paths is not None else None)

    def batch_problems(self, specs):
        """gmt_batch_create_problems: every problem's instance derived on the
        device (double-integrator problems from the shared Halton pool) into
        one solvable batch.  -> (Batch, status codes); the batch's query k is
        the k-th problem whose status is 0."""
        pb = specs if isinstance(specs, ProblemBatch) else ProblemBatch(specs)
        status = np.zeros(pb.count, np.int32)
        h = C.c_void_p()
        check(lib().gmt_batch_create_problems(self.h, pb.array, pb.count, abi.ptr(status, C.c_int32), C.byref(h)))
        ok = int((status == 0).sum())
        b = Batch(self, h, ok, [None] * ok)
        b._problems = pb
        return b, status

    def pool_info(self) -> dict:
        """The context's shared sample pool: points, edges, last build ms."""
        k, e, ms, fb = C.c_int32(), C.c_int64(), C.c_double(), C.c_int32()
        st = (C.c_double * 8)()
        check(lib().gmt_ctx_pool_info(self.h, C.byref(k), C.byref(e), C.byref(ms), C.byref(fb), st))
        return {"pool_size": k.value, "edges": e.value, "build_ms": ms.value, "last_fallbacks": fb.value,
                "stage_ms": list(st)}

    def run_trial(self, scenario, seed: int, path_cap: int = 100000):
        """run_trial (simulator.cpp:66-176) -> (TrialOutcome, path_travelled [k, dim])."""
        sc = scenario.flat()
        out = abi.TrialOutcome()
        path = np.zeros(path_cap * scenario.spec.dim)
        check(lib().gmt_run_trial(self.h, C.byref(sc), seed, C.byref(out), abi.ptr(path, C.c_double),
                                  path_cap))
        k = min(out.path_len, path_cap)
        return out, path[: k * scenario.spec.dim].reshape(k, scenario.spec.dim)

    def plan_host(self, spec, coords, goal_count, graph: Graph, init_index, lam, radius):
        coords = abi.f64(coords)
        buf = abi.PlanBuffers(coords.shape[0])
        sc = spec.scene()
        gv = graph.view()
        check(lib().gmt_plan_host(self.h, C.byref(sc), abi.ptr(coords, C.c_double), coords.shape[0],
                                  goal_count, C.byref(gv), init_index, lam, radius,
                                  C.byref(buf.out)))
        return buf.result()

    def batch(self, instances, lam: float = 1.0, init_index=None) -> Batch:
        arr = (C.c_void_p * len(instances))(*[i.h.value for i in instances])
        ii = None if init_index is None else abi.i32(init_index)
        h = C.c_void_p()
        check(lib().gmt_batch_create(self.h, len(instances), arr, abi.ptr(ii, C.c_int32), lam,
                                     C.byref(h)))
        return Batch(self, h, len(instances), [i.n for i in instances], instances)


class PinnedArray:
    """A numpy view of page-locked host memory from gmt_host_alloc."""

    def __init__(self, count: int, dtype):
        self.dtype = np.dtype(dtype)
        nbytes = max(int(count), 1) * self.dtype.itemsize
        self.p = C.c_void_p()
        check(lib().gmt_host_alloc(nbytes, C.byref(self.p)))
        buf = (C.c_char * nbytes).from_address(self.p.value)
        self.a = np.frombuffer(buf, dtype=self.dtype, count=max(int(count), 1))[: int(count)]

    def __del__(self):
        try:
            if self.p:
                lib().gmt_host_free(self.p)
                self.p = None
        except Exception:
            pass


class PackedBatch:
    """Independent Euclidean queries packed back to back in pinned host
    memory: the gmt_batch_host layout of include/gmt_b200.h.  `entries` are
    (spec, coords [n,d], goal_count, Graph, init_index) tuples."""

    def __init__(self, entries, want_tree: bool = True):
        self.count = len(entries)
        d = entries[0][0].dim
        ns = [e[1].shape[0] for e in entries]
        es = [e[3].num_edges for e in entries]
        bs = [e[0].num_boxes for e in entries]
        tn, te, tb = sum(ns), sum(es), sum(bs)
        A = PinnedArray
        self.node_off = A(self.count + 1, np.int64)
        self.edge_off = A(self.count + 1, np.int64)
        self.box_off = A(self.count + 1, np.int32)
        self.coords = A(tn * d, np.float64)
        self.box_lo = A(tb * d, np.float64)
        self.box_hi = A(tb * d, np.float64)
        self.goal_lo = A(self.count * d, np.float64)
        self.goal_hi = A(self.count * d, np.float64)
        self.row_ptr = A(tn + self.count, np.int64)
        self.col = A(te, np.int32)
        self.cost = A(te, np.float64)
        self.goal_count = A(self.count, np.int32)
        self.init_index = A(self.count, np.int32)
        self.radius = A(self.count, np.float64)
        self.node_off.a[:] = np.concatenate([[0], np.cumsum(ns)])
        self.edge_off.a[:] = np.concatenate([[0], np.cumsum(es)])
        self.box_off.a[:] = np.concatenate([[0], np.cumsum(bs)])
        for q, (spec, coords, gc, g, ii) in enumerate(entries):
            no, eo, bo = self.node_off.a[q], self.edge_off.a[q], self.box_off.a[q]
            n, nb = coords.shape[0], spec.num_boxes
            self.coords.a[no * d:(no + n) * d] = coords.reshape(-1)
            self.box_lo.a[bo * d:(bo + nb) * d] = spec.box_lo.reshape(-1)
            self.box_hi.a[bo * d:(bo + nb) * d] = spec.box_hi.reshape(-1)
            self.goal_lo.a[q * d:(q + 1) * d] = spec.goal_lo
            self.goal_hi.a[q * d:(q + 1) * d] = spec.goal_hi
            self.row_ptr.a[no + q:no + q + n + 1] = g.out_ptr
            self.col.a[eo:eo + g.num_edges] = g.out_col
            self.cost.a[eo:eo + g.num_edges] = g.out_cost
            self.goal_count.a[q] = gc
            self.init_index.a[q] = ii
            self.radius.a[q] = g.radius
        self.total_nodes, self.total_edges = tn, te
        self.paths = A(tn, np.int32)
        self.label = A(tn, np.uint8) if want_tree else None
        self.tree_cost = A(tn, np.float64) if want_tree else None
        self.parent = A(tn, np.int32) if want_tree else None
        self.iteration_added = A(tn, np.int64) if want_tree else None
        s = abi.BatchHost()
        s.count, s.dim = self.count, d
        for name, ct in (("node_off", C.c_int64), ("edge_off", C.c_int64), ("box_off", C.c_int32),
                         ("coords", C.c_double), ("box_lo", C.c_double), ("box_hi", C.c_double),
                         ("goal_lo", C.c_double), ("goal_hi", C.c_double),
                         ("row_ptr", C.c_int64), ("col", C.c_int32), ("cost", C.c_double),
                         ("goal_count", C.c_int32), ("init_index", C.c_int32),
                         ("radius", C.c_double)):
            setattr(s, name, abi.ptr(getattr(self, name).a, ct))
        self.struct = s
        self.summaries = (abi.PlanSummary * self.count)()

    @property
    def h2d_bytes(self) -> int:
        return sum(getattr(self, k).a.nbytes for k in (
            "coords", "box_lo", "box_hi", "goal_lo", "goal_hi", "row_ptr", "col", "cost"))

    @property
    def d2h_bytes(self) -> int:
        b = C.sizeof(abi.PlanSummary) * self.count + self.paths.a.nbytes
        for k in ("label", "tree_cost", "parent", "iteration_added"):
            if getattr(self, k) is not None:
                b += getattr(self, k).a.nbytes
        return b

    def query_result(self, q: int) -> abi.PlanResultPy:
        """PlanResult-shaped view of query q after a plan_batch_host call."""
        s = self.summaries[q]
        no, n1 = self.node_off.a[q], self.node_off.a[q + 1]
        t = (lambda x: None if x is None else x.a[no:n1].copy())
        return abi.PlanResultPy(status=s.status, cost=s.cost, iterations=s.iterations,
                                total_collision_checks=s.total_collision_checks,
                                path_indices=self.paths.a[no:no + s.path_len].copy(),
                                label=t(self.label), tree_cost=t(self.tree_cost),
                                parent=t(self.parent), iteration_added=t(self.iteration_added))


def plan_batch_host(ctx: Context, pb: PackedBatch, lam: float = 1.0):
    """gmt_plan_batch_host: H2D of the packed queries, one solve launch,
    D2H of summaries, paths and (if allocated) the trees."""
    opt = lambda x, ct: abi.ptr(None if x is None else x.a, ct)  # noqa: E731
    check(lib().gmt_plan_batch_host(ctx.h, C.byref(pb.struct), lam, pb.summaries,
                                    abi.ptr(pb.paths.a, C.c_int32), opt(pb.label, C.c_uint8),
                                    opt(pb.tree_cost, C.c_double), opt(pb.parent, C.c_int32),
                                    opt(pb.iteration_added, C.c_int64)))
    return pb.summaries


# ---- GMTG v1 graph cache (graph.cpp:190-343); host-only, no device needed ----
def problem_key(spec) -> int:
    """problem_key (problem.cpp:281-303) of a Euclidean problem."""
    k = C.c_uint64()
    p = spec.flat()
    check(lib().gmt_problem_key(C.byref(p), C.byref(k)))
    return k.value


def graph_cache_save(file: str, key: int, graph: Graph) -> None:
    """save_graph_cache (graph.cpp:240-276) of a host CSR graph."""
    check(lib().gmt_graph_cache_save(os.fsencode(file), key, graph.n, graph.radius,
                                     abi.ptr(graph.out_ptr, C.c_int64),
                                     abi.ptr(graph.out_col, C.c_int32),
                                     abi.ptr(graph.out_cost, C.c_double)))


def graph_cache_load(file: str, key: int, n: int, radius: float, dim: int = 0):
    """load_graph_cache (graph.cpp:278-343): the Graph, or None on a miss."""
    hit, ne = C.c_int32(), C.c_int64()
    z = lambda t: abi.ptr(None, t)  # noqa: E731
    check(lib().gmt_graph_cache_load(os.fsencode(file), key, n, radius, C.byref(hit), C.byref(ne), 0,
                                     z(C.c_int64), z(C.c_int32), z(C.c_double)))
    if not hit.value:
        return None
    E = ne.value
    ptr = np.zeros(n + 1, np.int64)
    col, cost = np.zeros(max(E, 1), np.int32), np.zeros(max(E, 1))
    check(lib().gmt_graph_cache_load(os.fsencode(file), key, n, radius, C.byref(hit), C.byref(ne), E,
                                     abi.ptr(ptr, C.c_int64), abi.ptr(col, C.c_int32),
                                     abi.ptr(cost, C.c_double)))
    if not hit.value:
        return None
    E = ne.value
    return Graph(n, radius, ptr, col[:E], cost[:E], dim=dim)


def _problem_file_spec(h):
    from . import problem as P
    v = abi.Problem()
    notes = C.c_char_p()
    try:
        check(lib().gmt_problem_file_view(h, C.byref(v), C.byref(notes)))
        d, nb = v.scene.dim, v.scene.num_boxes
        arr = lambda p, m: np.ctypeslib.as_array(p, shape=(m,)).copy() if m else np.zeros(0)  # noqa: E731
        spec = P.ProblemSpec(
            dim=d, box_lo=arr(v.scene.box_lo, nb * d).reshape(nb, d), box_hi=arr(v.scene.box_hi, nb * d).reshape(nb, d),
            goal_lo=arr(v.scene.goal_lo, d), goal_hi=arr(v.scene.goal_hi, d), init=arr(v.init, d), n=v.n,
            lam=v.lambda_, eta=v.eta, radius_override=v.radius_override if v.radius_override > 0.0 else None,
            sampling_kind=v.sampling.kind, start_index=v.sampling.start_index, seed=v.sampling.seed,
            notes=(notes.value or b"").decode("utf-8"), steering=v.steering)
        if v.steering == abi.STEER_DUBINS_AIRPLANE:
            spec.init_heading = v.init_heading if v.init_has_heading else None
            spec.dubins_rho = v.dubins.rho
            spec.dubins_step = v.dubins.discretization_step
            spec.dubins_planar = bool(v.dubins.planar_cost_only)
        return spec
    finally:
        lib().gmt_problem_file_destroy(h)


def parse_problem(text: str):
    """parse_problem (problem.cpp:102-223) through the C ABI
    (gmt_problem_parse) -> ProblemSpec; InvalidInputError with the
    reference's path-named message on any error."""
    data = text.encode("utf-8") if isinstance(text, str) else bytes(text)
    h = C.c_void_p()
    check(lib().gmt_problem_parse(data, len(data), C.byref(h)))
    return _problem_file_spec(h)


def load_problem(path: str):
    """load_problem (problem.cpp:225-231) through the C ABI."""
    h = C.c_void_p()
    check(lib().gmt_problem_load(os.fsencode(path), C.byref(h)))
    return _problem_file_spec(h)


def run_campaign(scenario, latencies, rates, sigmas, workers: int = 8, device: int = 0):
    """run_campaign (simulator.cpp:178-227) -> successes per cell, shape
    (len(latencies), len(rates), len(sigmas))."""
    sc = scenario.flat()
    lat, rat, sig = abi.f64(latencies), abi.f64(rates), abi.f64(sigmas)
    out = np.zeros(len(lat) * len(rat) * len(sig), np.int32)
    check(lib().gmt_run_campaign(device, C.byref(sc), abi.ptr(lat, C.c_double), len(lat),
                                 abi.ptr(rat, C.c_double), len(rat), abi.ptr(sig, C.c_double),
                                 len(sig), workers, abi.ptr(out, C.c_int32)))
    return out.reshape(len(lat), len(rat), len(sig))

