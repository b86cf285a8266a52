"""TEST INFRASTRUCTURE: the CPU oracle for the GMT* hot path.

Two interchangeable CPU implementations with one Python surface:

* ``port()``  -- liboracle.so, the plain-C restatement in gmt_oracle.c (every
  function cites the reference file:line it restates).
* ``ref()``   -- _ref/libgmtref.so, the UNMODIFIED reference gmtplan compiled
  from /root/reference/proj/src (see Makefile), wrapped by ref_capi.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
legs may import this package, and only as the checker or the timed CPU
baseline -- never as the product path.  The product library
(paper_1705_02403_b200) does not import it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_1705_02403_b200 import abi
from paper_1705_02403_b200.errors import raise_for

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libgmtref.so")

_dp = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_P = C.POINTER


def build(quiet: bool = True) -> None:
    """make -C oracle: the restatement always, the reference when
    /root/reference is present (building the checker is not using it)."""
    subprocess.run(["make", "-C", HERE, "-j8"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


class _Lib:
    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} is not built (run make -C oracle)")
        self.path = path
        self.prefix = prefix
        self.lib = C.CDLL(path)
        L = self.lib
        P = prefix

        def fn(name, restype, *argtypes):
            f = getattr(L, P + name)
            f.restype = restype
            f.argtypes = list(argtypes)
            return f

        self._last_error = fn("last_error", C.c_char_p)
        self._halton = fn("halton", C.c_int, C.c_uint64, C.c_uint32, _dp)
        self._nth_prime = fn("nth_prime", C.c_int, C.c_int, _P(C.c_uint32))
        self._point_free = fn("point_free", C.c_int, _P(abi.Scene), _dp, _i32p)
        self._segment_free = fn("segment_free", C.c_int, _P(abi.Scene), _dp, _dp, _i32p)
        self._sample_free = fn("sample_free", C.c_int, C.c_int32, _P(abi.Scene),
                               _P(abi.SampleSource), _dp, _dp, _i32p, _i32p)
        self._append_init = fn("append_init", C.c_int, C.c_int32, _dp, _dp, _i32p, _dp, C.c_int32,
                               C.c_double, _dp, _dp, _i32p, _i32p, _i32p)
        self._unit_ball = fn("unit_ball_volume", C.c_int, C.c_int32, _dp)
        self._radius = fn("connection_radius", C.c_int, C.c_int32, C.c_int64, C.c_double,
                          C.c_double, _dp)
        self._graph = fn("build_neighbor_graph", C.c_int, _dp, C.c_int32, C.c_int32, C.c_double,
                         C.c_int32, _i64p, _i64p, _i32p, _dp)
        self._plan = fn("gmt_plan", C.c_int, _P(abi.Scene), _dp, C.c_int32, C.c_int32,
                        _P(abi.GraphView), C.c_int32, C.c_double, C.c_double, C.c_int32,
                        _P(abi.PlanOut))
        self._fmt = fn("fmt_plan", C.c_int, _P(abi.Scene), _dp, C.c_int32, C.c_int32,
                       _P(abi.GraphView), C.c_int32, _P(abi.PlanOut))

    def _check(self, rc: int):
        if rc != 0:
            raise_for(rc, self._last_error().decode())

    # ---- sampling.cpp ------------------------------------------------------
    def halton(self, index: int, base: int) -> float:
        out = C.c_double()
        self._check(self._halton(index, base, C.byref(out)))
        return out.value

    def nth_prime(self, k: int) -> int:
        out = C.c_uint32()
        self._check(self._nth_prime(k, C.byref(out)))
        return out.value

    def point_free(self, spec, p) -> bool:
        p = abi.f64(p)
        out = C.c_int32()
        sc = spec.scene()
        self._check(self._point_free(C.byref(sc), abi.ptr(p, C.c_double), C.byref(out)))
        return bool(out.value)

    def segment_free(self, spec, a, b) -> bool:
        a, b = abi.f64(a), abi.f64(b)
        out = C.c_int32()
        sc = spec.scene()
        self._check(self._segment_free(C.byref(sc), abi.ptr(a, C.c_double), abi.ptr(b, C.c_double),
                                       C.byref(out)))
        return bool(out.value)

    def sample_free(self, spec, n: int | None = None):
        """-> (coords [n, dim], goal_indices)"""
        n = spec.n if n is None else n
        coords = np.zeros((n + 1) * spec.dim, np.float64)
        gidx = np.zeros(n + 1, np.int32)
        gcount = C.c_int32()
        sc, src = spec.scene(), spec.source()
        self._check(self._sample_free(n, C.byref(sc), C.byref(src), abi.ptr(coords, C.c_double),
                                      abi.ptr(None, C.c_double), abi.ptr(gidx, C.c_int32),
                                      C.byref(gcount)))
        return coords[: n * spec.dim].reshape(n, spec.dim), gidx[: gcount.value].copy()

    def append_init(self, coords: np.ndarray, goal_idx: np.ndarray, init, goal_lo, goal_hi):
        """-> (coords', goal_idx', init_index)"""
        n0, dim = coords.shape
        buf = np.zeros((n0 + 1) * dim, np.float64)
        buf[: n0 * dim] = coords.reshape(-1)
        g = np.zeros(n0 + 2, np.int32)
        g[: len(goal_idx)] = goal_idx
        n = C.c_int32(n0)
        gc = C.c_int32(len(goal_idx))
        idx = C.c_int32()
        init, gl, gh = abi.f64(init), abi.f64(goal_lo), abi.f64(goal_hi)
        self._check(self._append_init(dim, abi.ptr(buf, C.c_double), abi.ptr(None, C.c_double),
                                      C.byref(n), abi.ptr(init, C.c_double), 0, 0.0,
                                      abi.ptr(gl, C.c_double), abi.ptr(gh, C.c_double),
                                      abi.ptr(g, C.c_int32), C.byref(gc), C.byref(idx)))
        return buf[: n.value * dim].reshape(n.value, dim), g[: gc.value].copy(), idx.value

    # ---- graph.cpp ---------------------------------------------------------
    def unit_ball_volume(self, d: int) -> float:
        out = C.c_double()
        self._check(self._unit_ball(d, C.byref(out)))
        return out.value

    def connection_radius(self, dim: int, n: int, eta: float = 0.0, mu: float = 1.0) -> float:
        out = C.c_double()
        self._check(self._radius(dim, n, eta, mu, C.byref(out)))
        return out.value

    def build_neighbor_graph(self, coords: np.ndarray, radius: float, workers: int = 1):
        """-> (out_ptr int64[n+1], out_col int32[E], out_cost f64[E])"""
        coords = abi.f64(coords)
        n, dim = coords.shape
        ne = C.c_int64()
        self._check(self._graph(abi.ptr(coords, C.c_double), n, dim, radius, workers, C.byref(ne),
                                abi.ptr(None, C.c_int64), abi.ptr(None, C.c_int32),
                                abi.ptr(None, C.c_double)))
        ptr = np.zeros(n + 1, np.int64)
        col = np.zeros(max(ne.value, 1), np.int32)
        cost = np.zeros(max(ne.value, 1), np.float64)
        self._check(self._graph(abi.ptr(coords, C.c_double), n, dim, radius, workers, C.byref(ne),
                                abi.ptr(ptr, C.c_int64), abi.ptr(col, C.c_int32),
                                abi.ptr(cost, C.c_double)))
        return ptr, col[: ne.value].copy(), cost[: ne.value].copy()

    # ---- planner.cpp -------------------------------------------------------
    def gmt_plan(self, spec, coords, goal_count, graph, init_index, lam, radius, workers=1):
        coords = abi.f64(coords)
        n = coords.shape[0]
        buf = abi.PlanBuffers(n)
        sc = spec.scene()
        gv = graph.view()
        self._check(self._plan(C.byref(sc), abi.ptr(coords, C.c_double), n, goal_count,
                               C.byref(gv), init_index, lam, radius, workers, C.byref(buf.out)))
        return buf.result()

    def fmt_plan(self, spec, coords, goal_count, graph, init_index):
        coords = abi.f64(coords)
        n = coords.shape[0]
        buf = abi.PlanBuffers(n)
        sc = spec.scene()
        gv = graph.view()
        self._check(self._fmt(C.byref(sc), abi.ptr(coords, C.c_double), n, goal_count,
                              C.byref(gv), init_index, C.byref(buf.out)))
        return buf.result()


class PortLib(_Lib):
    """The C restatement, plus its statements of the NEW double-integrator
    and quadrotor models (no reference exists for them)."""

    def __init__(self):
        super().__init__(PORT_SO, "oracle_")
        L = self.lib
        L.oracle_di_cost.restype = C.c_double
        L.oracle_di_cost.argtypes = [_dp, _dp, C.c_double, C.c_double, _dp]
        L.oracle_di_coord.restype = C.c_double
        L.oracle_di_coord.argtypes = [_dp, _dp, C.c_double, C.c_int, C.c_int, C.c_int, C.c_double]
        L.oracle_di_paths.restype = None
        L.oracle_di_paths.argtypes = [_dp, C.c_int32, _i64p, _i32p, _dp, C.c_int, C.c_double, _dp]
        L.oracle_build_di_graph.restype = C.c_int
        L.oracle_build_di_graph.argtypes = [_dp, C.c_int32, C.c_double, C.c_double, C.c_double,
                                            _i64p, _i64p, _i32p, _dp, _dp]
        _qp = C.POINTER(abi.QuadParams)
        L.oracle_quad_cost.restype = C.c_double
        L.oracle_quad_cost.argtypes = [_dp, _dp, _qp, _dp]
        L.oracle_quad_coord.restype = C.c_double
        L.oracle_quad_coord.argtypes = [_dp, _dp, C.c_double, C.c_int, C.c_int, _qp]
        L.oracle_quad_paths.restype = None
        L.oracle_quad_paths.argtypes = [_dp, C.c_int32, _i64p, _i32p, _dp, _qp, _dp]
        L.oracle_build_quad_graph.restype = C.c_int
        L.oracle_build_quad_graph.argtypes = [_dp, C.c_int32, _qp, C.c_double, _i64p, _i64p, _i32p,
                                              _dp, _dp]

    def di_cost(self, x0, x1, vmax=0.5, weight=1.0):
        x0, x1 = abi.f64(x0), abi.f64(x1)
        t = C.c_double()
        c = self.lib.oracle_di_cost(abi.ptr(x0, C.c_double), abi.ptr(x1, C.c_double), vmax, weight,
                                    C.byref(t))
        return c, t.value

    def di_waypoints(self, x0, x1, tau, segments=8, vmax=0.5):
        x0, x1 = abi.f64(x0), abi.f64(x1)
        return np.array([[self.lib.oracle_di_coord(abi.ptr(x0, C.c_double), abi.ptr(x1, C.c_double),
                                                   tau, k, i, segments, vmax) for i in range(6)]
                         for k in range(segments + 1)])

    def build_di_graph(self, coords, radius, vmax=0.5, weight=1.0):
        """-> (out_ptr, out_col, out_cost, out_tau)"""
        coords = abi.f64(coords)
        n = coords.shape[0]
        ne = C.c_int64()
        self._check(self.lib.oracle_build_di_graph(abi.ptr(coords, C.c_double), n, vmax, weight,
                                                   radius, C.byref(ne), abi.ptr(None, C.c_int64),
                                                   abi.ptr(None, C.c_int32),
                                                   abi.ptr(None, C.c_double),
                                                   abi.ptr(None, C.c_double)))
        E = ne.value
        ptr = np.zeros(n + 1, np.int64)
        col = np.zeros(max(E, 1), np.int32)
        cost, tau = np.zeros(max(E, 1)), np.zeros(max(E, 1))
        self._check(self.lib.oracle_build_di_graph(abi.ptr(coords, C.c_double), n, vmax, weight,
                                                   radius, C.byref(ne), abi.ptr(ptr, C.c_int64),
                                                   abi.ptr(col, C.c_int32),
                                                   abi.ptr(cost, C.c_double),
                                                   abi.ptr(tau, C.c_double)))
        return ptr, col[:E], cost[:E], tau[:E]

    def di_graph(self, coords, radius, segments=8, vmax=0.5, weight=1.0):
        """Reference-shaped directed Graph with cached waypoint paths (path
        ids = out-edge indices, in-lists by ascending source)."""
        from paper_1705_02403_b200.graph import Graph
        ptr, col, cost, tau = self.build_di_graph(coords, radius, vmax, weight)
        n, E, M1 = coords.shape[0], len(col), segments + 1
        pts = np.zeros((max(E, 1), M1, 6))
        coords = abi.f64(coords)
        self.lib.oracle_di_paths(abi.ptr(coords, C.c_double), n, abi.ptr(ptr, C.c_int64),
                                 abi.ptr(abi.i32(col), C.c_int32), abi.ptr(abi.f64(tau), C.c_double),
                                 segments, vmax, abi.ptr(pts, C.c_double))
        g = Graph(n, radius, ptr, col, cost, dim=6, directed=True,
                  out_path=np.arange(E, dtype=np.int32),
                  path_ptr=np.arange(E + 1, dtype=np.int64) * M1,
                  path_pts=pts[:E].reshape(-1))
        in_ptr, in_col, in_cost, in_path = g.transpose()
        g.in_ptr, g.in_col, g.in_cost, g.in_path = (abi.i64(in_ptr), abi.i32(in_col),
                                                     abi.f64(in_cost), abi.i32(in_path))
        g.out_tau = tau
        return g

    # ---- 12D quadrotor (NEW model) ----
    def quad_cost(self, x0, x1, params):
        x0, x1 = abi.f64(x0), abi.f64(x1)
        t = C.c_double()
        c = self.lib.oracle_quad_cost(abi.ptr(x0, C.c_double), abi.ptr(x1, C.c_double),
                                      C.byref(params), C.byref(t))
        return c, t.value

    def quad_waypoints(self, x0, x1, tau, params):
        x0, x1 = abi.f64(x0), abi.f64(x1)
        return np.array([[self.lib.oracle_quad_coord(abi.ptr(x0, C.c_double),
                                                     abi.ptr(x1, C.c_double), tau, k, i,
                                                     C.byref(params)) for i in range(12)]
                         for k in range(params.segments + 1)])

    def build_quad_graph(self, coords, radius, params):
        """-> (out_ptr, out_col, out_cost, out_tau)"""
        coords = abi.f64(coords)
        n = coords.shape[0]
        ne = C.c_int64()
        self._check(self.lib.oracle_build_quad_graph(abi.ptr(coords, C.c_double), n, C.byref(params),
                                                     radius, C.byref(ne), abi.ptr(None, C.c_int64),
                                                     abi.ptr(None, C.c_int32),
                                                     abi.ptr(None, C.c_double),
                                                     abi.ptr(None, C.c_double)))
        E = ne.value
        ptr = np.zeros(n + 1, np.int64)
        col = np.zeros(max(E, 1), np.int32)
        cost, tau = np.zeros(max(E, 1)), np.zeros(max(E, 1))
        self._check(self.lib.oracle_build_quad_graph(abi.ptr(coords, C.c_double), n, C.byref(params),
                                                     radius, C.byref(ne), abi.ptr(ptr, C.c_int64),
                                                     abi.ptr(col, C.c_int32),
                                                     abi.ptr(cost, C.c_double),
                                                     abi.ptr(tau, C.c_double)))
        return ptr, col[:E], cost[:E], tau[:E]

    def quad_graph(self, coords, radius, params):
        """As di_graph, for the quadrotor."""
        from paper_1705_02403_b200.graph import Graph
        ptr, col, cost, tau = self.build_quad_graph(coords, radius, params)
        n, E, M1 = coords.shape[0], len(col), params.segments + 1
        pts = np.zeros((max(E, 1), M1, 12))
        coords = abi.f64(coords)
        self.lib.oracle_quad_paths(abi.ptr(coords, C.c_double), n, abi.ptr(ptr, C.c_int64),
                                   abi.ptr(abi.i32(col), C.c_int32), abi.ptr(abi.f64(tau), C.c_double),
                                   C.byref(params), abi.ptr(pts, C.c_double))
        g = Graph(n, radius, ptr, col, cost, dim=12, directed=True,
                  out_path=np.arange(E, dtype=np.int32),
                  path_ptr=np.arange(E + 1, dtype=np.int64) * M1,
                  path_pts=pts[:E].reshape(-1))
        in_ptr, in_col, in_cost, in_path = g.transpose()
        g.in_ptr, g.in_col, g.in_cost, g.in_path = (abi.i64(in_ptr), abi.i32(in_col),
                                                     abi.f64(in_cost), abi.i32(in_path))
        g.out_tau = tau
        return g


class RefLib(_Lib):
    """The unmodified reference (plus its test-support oracles)."""

    def __init__(self):
        super().__init__(REF_SO, "ref_")
        L = self.lib
        L.ref_dijkstra_oracle.restype = C.c_int
        L.ref_dijkstra_oracle.argtypes = [_P(abi.Scene), _dp, C.c_int32, C.c_int32,
                                          _P(abi.GraphView), C.c_int32, _P(abi.PlanOut)]
        L.ref_instance_build.restype = C.c_int
        L.ref_instance_build.argtypes = [_P(abi.Problem), C.c_int32, _P(C.c_void_p)]
        L.ref_instance_build_many.restype = C.c_int
        L.ref_instance_build_many.argtypes = [_P(abi.Problem), C.c_int32, C.c_int32,
                                              _P(C.c_void_p)]
        L.ref_instance_destroy.restype = None
        L.ref_instance_destroy.argtypes = [C.c_void_p]
        L.ref_instance_info.restype = C.c_int
        L.ref_instance_info.argtypes = [C.c_void_p, _i32p, _i32p, _dp, _i64p, _i32p]
        L.ref_instance_download.restype = C.c_int
        L.ref_instance_download.argtypes = [C.c_void_p, _dp, _i32p, _i64p, _i32p, _dp]
        L.ref_dubins_costs.restype = C.c_int
        L.ref_dubins_costs.argtypes = [_dp, _dp, C.c_int64, C.c_int32, _P(abi.DubinsParams), _dp, _i32p]
        L.ref_instance_download_paths.restype = C.c_int
        L.ref_instance_download_paths.argtypes = [C.c_void_p, _i64p, _i32p, _dp, _i32p, _i32p, _i64p, _dp,
                                                  _i64p, _i64p]
        L.ref_run_trial.restype = C.c_int
        L.ref_run_trial.argtypes = [_P(abi.Scenario), C.c_uint64, _P(abi.TrialOutcome), _dp, C.c_int64]
        L.ref_run_campaign.restype = C.c_int
        L.ref_run_campaign.argtypes = [_P(abi.Scenario), _dp, C.c_int32, _dp, C.c_int32, _dp, C.c_int32,
                                       C.c_int32, _i32p]
        L.ref_problem_key.restype = C.c_int
        L.ref_problem_key.argtypes = [_P(abi.Problem), _P(C.c_uint64)]
        L.ref_instance_build_cached.restype = C.c_int
        L.ref_instance_build_cached.argtypes = [_P(abi.Problem), C.c_char_p, _P(C.c_void_p)]
        L.ref_save_graph_cache.restype = C.c_int
        L.ref_save_graph_cache.argtypes = [C.c_void_p, C.c_char_p, C.c_uint64, _i32p]
        L.ref_load_graph_cache.restype = C.c_int
        L.ref_load_graph_cache.argtypes = [C.c_char_p, C.c_uint64, _dp, C.c_int32, C.c_int32,
                                           C.c_double, _i32p, _i64p, _i64p, _i32p, _dp]
        L.ref_instance_plan.restype = C.c_int
        L.ref_instance_plan.argtypes = [C.c_void_p, C.c_double, C.c_int32, _P(abi.PlanOut)]
        L.ref_instance_time_plans.restype = C.c_int
        L.ref_instance_time_plans.argtypes = [C.c_void_p, C.c_double, C.c_int32, C.c_int32, _dp]
        L.ref_time_gmt_plan.restype = C.c_int
        L.ref_time_gmt_plan.argtypes = [_P(abi.Scene), _dp, C.c_int32, C.c_int32, _P(abi.GraphView), C.c_int32,
                                        C.c_double, C.c_double, C.c_int32, C.c_int32, _dp]
        L.ref_plan_many.restype = C.c_int
        L.ref_plan_many.argtypes = [_P(C.c_void_p), C.c_int32, C.c_double, C.c_int32,
                                    _P(abi.PlanSummary), _dp]
        L.ref_rng_create.restype = C.c_void_p
        L.ref_rng_create.argtypes = [C.c_uint64]
        L.ref_rng_destroy.restype = None
        L.ref_rng_destroy.argtypes = [C.c_void_p]
        L.ref_rng_next_u32.restype = C.c_uint32
        L.ref_rng_next_u32.argtypes = [C.c_void_p]
        L.ref_random_problem_new.restype = C.c_int
        L.ref_random_problem_new.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                             C.c_int32, _P(C.c_void_p)]
        L.ref_random_problem_free.restype = None
        L.ref_random_problem_free.argtypes = [C.c_void_p]
        L.ref_random_problem_info.restype = C.c_int
        L.ref_random_problem_info.argtypes = [C.c_void_p, _i32p, _i32p, _i32p, _dp, _i32p,
                                              _P(C.c_uint64)]
        L.ref_random_problem_get.restype = C.c_int
        L.ref_random_problem_get.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp, _dp, _i32p]
        L.ref_parse_problem.restype = C.c_int
        L.ref_parse_problem.argtypes = [C.c_char_p, _i32p, _i32p, _dp, _dp, _dp, _dp, _dp, _i32p,
                                        _dp, _dp, _dp, _i32p, _P(C.c_uint64), _P(C.c_uint64),
                                        _P(C.c_uint64), _i32p]

    def segment_free_many(self, spec, a, b) -> np.ndarray:
        """segment_free (space.cpp:80-90) of every row pair a[i] -> b[i]."""
        a, b = abi.f64(a), abi.f64(b)
        out = np.zeros(a.shape[0], np.uint8)
        sc = spec.scene()
        f = self.lib.ref_segment_free_many
        f.restype = C.c_int
        f.argtypes = [_P(abi.Scene), _dp, _dp, C.c_int64, _P(C.c_uint8)]
        self._check(f(C.byref(sc), abi.ptr(a, C.c_double), abi.ptr(b, C.c_double), a.shape[0],
                      abi.ptr(out, C.c_uint8)))
        return out

    def time_gmt_plan(self, spec, coords, goal_count, graph, init_index, lam, radius, workers, reps):
        """Per-call ms of `reps` gmt_plan calls on an injected graph (timed in C)."""
        coords = abi.f64(coords)
        ms = np.zeros(reps)
        sc = spec.scene()
        gv = graph.view()
        self._check(self.lib.ref_time_gmt_plan(C.byref(sc), abi.ptr(coords, C.c_double), coords.shape[0],
                                               goal_count, C.byref(gv), init_index, lam, radius, workers,
                                               reps, abi.ptr(ms, C.c_double)))
        return ms

    def dijkstra_oracle(self, spec, coords, goal_count, graph, init_index):
        coords = abi.f64(coords)
        n = coords.shape[0]
        buf = abi.PlanBuffers(n)
        sc = spec.scene()
        gv = graph.view()
        self._check(self.lib.ref_dijkstra_oracle(C.byref(sc), abi.ptr(coords, C.c_double), n,
                                                 goal_count, C.byref(gv), init_index,
                                                 C.byref(buf.out)))
        return buf.result()

    # ---- ProblemInstance handles (build_instance, problem.cpp:336-363) ------
    def instance_build(self, spec, workers: int = 1) -> "RefInstance":
        h = C.c_void_p()
        p = spec.flat()
        self._check(self.lib.ref_instance_build(C.byref(p), workers, C.byref(h)))
        return RefInstance(self, h)

    def dubins_costs(self, x0s, x1s, dim: int, params):
        x0s = abi.f64(x0s).reshape(-1, dim + 1)
        x1s = abi.f64(x1s).reshape(-1, dim + 1)
        m = x0s.shape[0]
        cost, segs = np.zeros(m), np.zeros(m, np.int32)
        self._check(self.lib.ref_dubins_costs(abi.ptr(x0s, C.c_double), abi.ptr(x1s, C.c_double), m, dim,
                                              C.byref(params), abi.ptr(cost, C.c_double),
                                              abi.ptr(segs, C.c_int32)))
        return cost, segs

    # ---- simulator (simulator.cpp:66-227) ----------------------------------
    def run_trial(self, scenario, seed: int, path_cap: int = 100000):
        sc = scenario.flat()
        out = abi.TrialOutcome()
        path = np.zeros(path_cap * scenario.spec.dim)
        self._check(self.lib.ref_run_trial(C.byref(sc), seed, C.byref(out), abi.ptr(path, C.c_double),
                                           path_cap))
        k = min(out.path_len, path_cap)
        return out, path[: k * scenario.spec.dim].reshape(k, scenario.spec.dim)

    def run_campaign(self, scenario, latencies, rates, sigmas, workers: int = 8):
        sc = scenario.flat()
        lat, rat, sig = abi.f64(latencies), abi.f64(rates), abi.f64(sigmas)
        out = np.zeros(len(lat) * len(rat) * len(sig), np.int32)
        self._check(self.lib.ref_run_campaign(C.byref(sc), abi.ptr(lat, C.c_double), len(lat),
                                              abi.ptr(rat, C.c_double), len(rat),
                                              abi.ptr(sig, C.c_double), len(sig), workers,
                                              abi.ptr(out, C.c_int32)))
        return out.reshape(len(lat), len(rat), len(sig))

    # ---- graph cache (graph.cpp:190-343) and problem_key (problem.cpp:281-303)
    def problem_key(self, spec) -> int:
        k = C.c_uint64()
        p = spec.flat()
        self._check(self.lib.ref_problem_key(C.byref(p), C.byref(k)))
        return k.value

    def instance_build_cached(self, spec, cache_file: str) -> "RefInstance":
        h = C.c_void_p()
        p = spec.flat()
        self._check(self.lib.ref_instance_build_cached(C.byref(p), os.fsencode(cache_file), C.byref(h)))
        return RefInstance(self, h)

    def load_graph_cache(self, file: str, key: int, coords, radius: float):
        """-> (out_ptr, out_col, out_cost) or None on a miss."""
        coords = abi.f64(coords)
        n, dim = coords.shape
        hit, ne = C.c_int32(), C.c_int64()
        z = lambda t: abi.ptr(None, t)  # noqa: E731
        self._check(self.lib.ref_load_graph_cache(os.fsencode(file), key, abi.ptr(coords, C.c_double),
                                                  n, dim, radius, C.byref(hit), C.byref(ne),
                                                  z(C.c_int64), z(C.c_int32), z(C.c_double)))
        if not hit.value:
            return None
        E = ne.value
        ptr = np.zeros(n + 1, np.int64)
        col, cost = np.zeros(max(E, 1), np.int32), np.zeros(max(E, 1))
        self._check(self.lib.ref_load_graph_cache(os.fsencode(file), key, abi.ptr(coords, C.c_double),
                                                  n, dim, radius, C.byref(hit), C.byref(ne),
                                                  abi.ptr(ptr, C.c_int64), abi.ptr(col, C.c_int32),
                                                  abi.ptr(cost, C.c_double)))
        return ptr, col[:E], cost[:E]

    def di_pool(self, start_index: int, K: int, di, radius: float, threads: int):
        """Shared-pool rows of the double integrator (the oracle's C statement
        of the model) for the reference arm's DI instances."""
        f = self.lib.ref_di_pool_create
        f.restype = C.c_void_p
        f.argtypes = [C.c_uint64, C.c_int32, _P(abi.DiParams), C.c_double, C.c_int32]
        h = f(start_index, K, C.byref(di), radius, threads)
        return DiPoolRef(self, h)

    def di_instances(self, pool: "DiPoolRef", specs, threads: int):
        """Reference instances of DI problems: the reference's own sample_free
        and append_init, the DI graph from the pool rows + direct rows of the
        non-pool vertices, every edge's waypoint polyline cached."""
        arr = (abi.Problem * len(specs))(*[s.flat() for s in specs])
        hs = (C.c_void_p * len(specs))()
        f = self.lib.ref_di_pool_instances
        f.restype = C.c_int
        f.argtypes = [C.c_void_p, _P(abi.Problem), C.c_int32, C.c_int32, _P(C.c_void_p)]
        self._check(f(pool.h, arr, len(specs), threads, hs))
        return [RefInstance(self, C.c_void_p(h)) for h in hs]

    def instance_build_many(self, specs, threads: int):
        arr = (abi.Problem * len(specs))(*[s.flat() for s in specs])
        hs = (C.c_void_p * len(specs))()
        self._check(self.lib.ref_instance_build_many(arr, len(specs), threads, hs))
        return [RefInstance(self, C.c_void_p(h)) for h in hs]

    def plan_many(self, insts, lam: float, threads: int):
        hs = (C.c_void_p * len(insts))(*[i.h.value for i in insts])
        out = (abi.PlanSummary * len(insts))()
        sec = C.c_double()
        self._check(self.lib.ref_plan_many(hs, len(insts), lam, threads, out, C.byref(sec)))
        return list(out), sec.value

    # ---- the reference's own random problems (oracles.cpp:258-327) --------
    def rng(self, seed: int):
        return RefRng(self, seed)

    def random_problem(self, rng: "RefRng", dim=2, with_obstacles=True, n_min=120, n_max=350):
        h = C.c_void_p()
        self._check(self.lib.ref_random_problem_new(rng.h, dim, int(with_obstacles), n_min, n_max,
                                                    C.byref(h)))
        try:
            nb, ns, ii, gc = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
            r = C.c_double()
            sd = C.c_uint64()
            self._check(self.lib.ref_random_problem_info(h, C.byref(nb), C.byref(ns), C.byref(ii),
                                                         C.byref(r), C.byref(gc), C.byref(sd)))
            lo = np.zeros(max(nb.value, 1) * dim)
            hi = np.zeros(max(nb.value, 1) * dim)
            gl, gh, init = np.zeros(dim), np.zeros(dim), np.zeros(dim)
            coords = np.zeros(ns.value * dim)
            gidx = np.zeros(max(gc.value, 1), np.int32)
            self._check(self.lib.ref_random_problem_get(
                h, abi.ptr(lo, C.c_double), abi.ptr(hi, C.c_double), abi.ptr(gl, C.c_double),
                abi.ptr(gh, C.c_double), abi.ptr(init, C.c_double), abi.ptr(coords, C.c_double),
                abi.ptr(gidx, C.c_int32)))
        finally:
            self.lib.ref_random_problem_free(h)
        from paper_1705_02403_b200.problem import ProblemSpec
        spec = ProblemSpec(dim=dim, box_lo=lo[: nb.value * dim].reshape(-1, dim),
                           box_hi=hi[: nb.value * dim].reshape(-1, dim), goal_lo=gl, goal_hi=gh,
                           init=init, n=ns.value - 1 if ii.value == ns.value - 1 else ns.value)
        return dict(spec=spec, coords=coords.reshape(ns.value, dim), goal_idx=gidx[: gc.value],
                    init_index=ii.value, radius=r.value)

    def parse_problem(self, text: str):
        d, nb = C.c_int32(), C.c_int32()
        z = abi.ptr(None, C.c_double)
        zi = abi.ptr(None, C.c_int32)
        zu = C.cast(None, _P(C.c_uint64))
        self._check(self.lib.ref_parse_problem(text.encode(), C.byref(d), C.byref(nb), z, z, z, z,
                                               z, zi, z, z, z, zi, zu, zu, zu, zi))
        dim = d.value
        lo, hi = np.zeros(max(nb.value, 1) * dim), np.zeros(max(nb.value, 1) * dim)
        gl, gh, init = np.zeros(dim), np.zeros(dim), np.zeros(dim)
        n, kind, sk = C.c_int32(), C.c_int32(), C.c_int32()
        lam, eta, ro = C.c_double(), C.c_double(), C.c_double()
        si, seed, key = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self._check(self.lib.ref_parse_problem(
            text.encode(), C.byref(d), C.byref(nb), abi.ptr(lo, C.c_double),
            abi.ptr(hi, C.c_double), abi.ptr(gl, C.c_double), abi.ptr(gh, C.c_double),
            abi.ptr(init, C.c_double), C.byref(n), C.byref(lam), C.byref(eta), C.byref(ro),
            C.byref(kind), C.byref(si), C.byref(seed), C.byref(key), C.byref(sk)))
        return dict(dim=dim, box_lo=lo[: nb.value * dim].reshape(-1, dim),
                    box_hi=hi[: nb.value * dim].reshape(-1, dim), goal_lo=gl, goal_hi=gh,
                    init=init, n=n.value, lam=lam.value, eta=eta.value,
                    radius_override=ro.value or None, sampling_kind=kind.value,
                    start_index=si.value, seed=seed.value, key=key.value, steering=sk.value)


class DiPoolRef:
    def __init__(self, lib: "RefLib", h):
        self.lib, self.h = lib, h

    def __del__(self):
        try:
            f = self.lib.lib.ref_di_pool_destroy
            f.restype = None
            f.argtypes = [C.c_void_p]
            f(self.h)
        except Exception:
            pass


class RefRng:
    def __init__(self, lib: RefLib, seed: int):
        self.lib = lib
        self.h = C.c_void_p(lib.lib.ref_rng_create(seed))

    def next_u32(self) -> int:
        return self.lib.lib.ref_rng_next_u32(self.h)

    def __del__(self):
        try:
            self.lib.lib.ref_rng_destroy(self.h)
        except Exception:
            pass


class RefInstance:
    def __init__(self, lib: RefLib, h):
        self.lib = lib
        self.h = h

    def graph(self, dim: int):
        """The instance's NeighborGraph as a Graph with in-rows and cached
        edge paths (directed Dubins graphs)."""
        from paper_1705_02403_b200.graph import Graph
        info = self.info()
        n, E = info["n"], info["num_edges"]
        coords, gidx, optr, ocol, ocost = self.download(dim)
        npaths, npts = C.c_int64(), C.c_int64()
        z = lambda t: abi.ptr(None, t)  # noqa: E731
        self.lib._check(self.lib.lib.ref_instance_download_paths(self.h, z(C.c_int64), z(C.c_int32),
                                                                 z(C.c_double), z(C.c_int32),
                                                                 z(C.c_int32), z(C.c_int64),
                                                                 z(C.c_double), C.byref(npaths),
                                                                 C.byref(npts)))
        iptr, icol, icost = np.zeros(n + 1, np.int64), np.zeros(max(E, 1), np.int32), np.zeros(max(E, 1))
        ipath, opath = np.zeros(max(E, 1), np.int32), np.zeros(max(E, 1), np.int32)
        pptr = np.zeros(npaths.value + 1, np.int64)
        pts = np.zeros(max(npts.value, 1) * dim)
        self.lib._check(self.lib.lib.ref_instance_download_paths(
            self.h, abi.ptr(iptr, C.c_int64), abi.ptr(icol, C.c_int32), abi.ptr(icost, C.c_double),
            abi.ptr(ipath, C.c_int32), abi.ptr(opath, C.c_int32), abi.ptr(pptr, C.c_int64),
            abi.ptr(pts, C.c_double), C.byref(npaths), C.byref(npts)))
        g = Graph(n, info["radius"], optr, ocol, ocost, dim=dim, directed=True, in_ptr=iptr,
                  in_col=icol[:E], in_cost=icost[:E], out_path=opath[:E], in_path=ipath[:E],
                  path_ptr=pptr, path_pts=pts[: npts.value * dim])
        return coords, gidx, g

    def save_cache(self, file: str, key: int) -> bool:
        ok = C.c_int32()
        self.lib._check(self.lib.lib.ref_save_graph_cache(self.h, os.fsencode(file), key, C.byref(ok)))
        return bool(ok.value)

    def info(self):
        n, ii, gc = C.c_int32(), C.c_int32(), C.c_int32()
        r = C.c_double()
        ne = C.c_int64()
        self.lib._check(self.lib.lib.ref_instance_info(self.h, C.byref(n), C.byref(ii), C.byref(r),
                                                       C.byref(ne), C.byref(gc)))
        return dict(n=n.value, init_index=ii.value, radius=r.value, num_edges=ne.value,
                    goal_count=gc.value)

    def download(self, dim: int):
        inf = self.info()
        n, ne = inf["n"], inf["num_edges"]
        coords = np.zeros(n * dim)
        gidx = np.zeros(max(inf["goal_count"], 1), np.int32)
        ptr = np.zeros(n + 1, np.int64)
        col = np.zeros(max(ne, 1), np.int32)
        cost = np.zeros(max(ne, 1))
        self.lib._check(self.lib.lib.ref_instance_download(
            self.h, abi.ptr(coords, C.c_double), abi.ptr(gidx, C.c_int32), abi.ptr(ptr, C.c_int64),
            abi.ptr(col, C.c_int32), abi.ptr(cost, C.c_double)))
        return coords.reshape(n, dim), gidx[: inf["goal_count"]], ptr, col[:ne], cost[:ne]

    def time_plans(self, lam: float, workers: int, reps: int):
        """Per-call ms of `reps` gmt_plan calls on this instance (timed in C)."""
        ms = np.zeros(reps)
        self.lib._check(self.lib.lib.ref_instance_time_plans(self.h, lam, workers, reps, abi.ptr(ms, C.c_double)))
        return ms

    def plan(self, lam: float, workers: int = 1):
        n = self.info()["n"]
        buf = abi.PlanBuffers(n)
        self.lib._check(self.lib.lib.ref_instance_plan(self.h, lam, workers, C.byref(buf.out)))
        return buf.result()

    def __del__(self):
        try:
            if self.h:
                self.lib.lib.ref_instance_destroy(self.h)
                self.h = None
        except Exception:
            pass


_port = None
_ref = None


def port() -> PortLib:
    global _port
    if _port is None:
        _port = PortLib()
    return _port


def ref() -> RefLib:
    global _ref
    if _ref is None:
        _ref = RefLib()
    return _ref


def ref_available() -> bool:
    return os.path.exists(REF_SO)
