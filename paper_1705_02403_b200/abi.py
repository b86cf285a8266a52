"""ctypes mirror of include/gmt_b200.h (the C ABI of the B200 GMT* planner).

Only struct layouts and helpers that turn numpy arrays into the flat views
live here; the loaders for the product library (``_native``) and for the
oracle libraries (``oracle/``) both use these definitions so the same Python
objects can be handed to either implementation.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

GMT_OK = 0
GMT_E_INVALID_INPUT = 1
GMT_E_INFEASIBLE_SAMPLING = 2
GMT_E_GOAL_BLOCKED = 3
GMT_E_CUDA = 4
GMT_E_NO_DEVICE = 5
GMT_E_INTERNAL = 6

PLAN_SUCCESS = 0
PLAN_FAILURE_OPEN_EMPTY = 1
PLAN_INFEASIBLE_INPUT = 2

LABEL_UNEXPLORED = 0
LABEL_OPEN = 1
LABEL_CLOSED = 2

SAMPLE_HALTON = 0
SAMPLE_UNIFORM = 1

_dp = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u8p = C.POINTER(C.c_uint8)


class Scene(C.Structure):
    _fields_ = [
        ("dim", C.c_int32),
        ("num_boxes", C.c_int32),
        ("box_lo", _dp),
        ("box_hi", _dp),
        ("goal_lo", _dp),
        ("goal_hi", _dp),
    ]


class SampleSource(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("with_heading", C.c_int32),
        ("start_index", C.c_uint64),
        ("seed", C.c_uint64),
    ]


class GraphView(C.Structure):
    _fields_ = [
        ("n", C.c_int32),
        ("dim", C.c_int32),
        ("radius", C.c_double),
        ("directed", C.c_int32),
        ("reserved", C.c_int32),
        ("out_ptr", _i64p),
        ("out_col", _i32p),
        ("out_cost", _dp),
        ("out_path", _i32p),
        ("in_ptr", _i64p),
        ("in_col", _i32p),
        ("in_cost", _dp),
        ("in_path", _i32p),
        ("num_paths", C.c_int64),
        ("path_ptr", _i64p),
        ("path_pts", _dp),
    ]


class PlanOut(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("goal_node", C.c_int32),
        ("cost", C.c_double),
        ("iterations", C.c_int64),
        ("total_collision_checks", C.c_int64),
        ("path_len", C.c_int32),
        ("num_stats", C.c_int32),
        ("tree_size", C.c_int32),
        ("stats_cap", C.c_int32),
        ("path", _i32p),
        ("label", _u8p),
        ("tree_cost", _dp),
        ("parent", _i32p),
        ("iteration_added", _i64p),
        ("group_sizes", _i32p),
        ("nodes_added", _i32p),
        ("collision_checks", _i64p),
    ]


class PlanSummary(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("goal_node", C.c_int32),
        ("cost", C.c_double),
        ("iterations", C.c_int64),
        ("total_collision_checks", C.c_int64),
        ("path_len", C.c_int32),
        ("num_stats", C.c_int32),
    ]


STEER_EUCLIDEAN = 0
STEER_DUBINS_AIRPLANE = 1
STEER_DOUBLE_INTEGRATOR = 2
STEER_QUADROTOR = 3


class DiParams(C.Structure):
    """gmt_di_params: 6D double integrator (NEW model)."""
    _fields_ = [
        ("vmax", C.c_double),
        ("weight", C.c_double),
        ("segments", C.c_int32),
        ("reserved", C.c_int32),
    ]


class QuadParams(C.Structure):
    """gmt_quad_params: 12D linearised quadrotor (NEW model)."""
    _fields_ = [
        ("g", C.c_double),
        ("vmax", C.c_double),
        ("amax", C.c_double),
        ("ymax", C.c_double),
        ("wmax", C.c_double),
        ("weight", C.c_double),
        ("segments", C.c_int32),
        ("reserved", C.c_int32),
    ]


class DubinsParams(C.Structure):
    """gmt_dubins_params (SteeringModel, steering.hpp:9-23)."""
    _fields_ = [
        ("rho", C.c_double),
        ("discretization_step", C.c_double),
        ("planar_cost_only", C.c_int32),
        ("reserved", C.c_int32),
    ]


class Problem(C.Structure):
    _fields_ = [
        ("scene", Scene),
        ("init", _dp),
        ("init_has_heading", C.c_int32),
        ("init_heading", C.c_double),
        ("n", C.c_int32),
        ("lambda_", C.c_double),
        ("eta", C.c_double),
        ("radius_override", C.c_double),
        ("sampling", SampleSource),
        ("steering", C.c_int32),
        ("reserved", C.c_int32),
        ("di", DiParams),
        ("quad", QuadParams),
        ("dubins", DubinsParams),
    ]


class BatchHost(C.Structure):
    _fields_ = [
        ("count", C.c_int32),
        ("dim", C.c_int32),
        ("node_off", _i64p),
        ("edge_off", _i64p),
        ("box_off", _i32p),
        ("coords", _dp),
        ("box_lo", _dp),
        ("box_hi", _dp),
        ("goal_lo", _dp),
        ("goal_hi", _dp),
        ("row_ptr", _i64p),
        ("col", _i32p),
        ("cost", _dp),
        ("goal_count", _i32p),
        ("init_index", _i32p),
        ("radius", _dp),
    ]


def ptr(a: np.ndarray | None, ctype):
    """Pointer to a contiguous numpy array (or NULL)."""
    if a is None:
        return C.cast(None, C.POINTER(ctype))
    assert a.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    return a.ctypes.data_as(C.POINTER(ctype))


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


class PlanBuffers:
    """Caller-owned output arrays for one PlanOut of an n-node problem."""

    def __init__(self, n: int, want_tree: bool = True, want_stats: bool = True):
        self.n = n
        self.path = np.zeros(max(n, 1), np.int32)
        self.label = np.zeros(max(n, 1), np.uint8) if want_tree else None
        self.tree_cost = np.zeros(max(n, 1), np.float64) if want_tree else None
        self.parent = np.zeros(max(n, 1), np.int32) if want_tree else None
        self.iteration_added = np.zeros(max(n, 1), np.int64) if want_tree else None
        cap = n + 2
        self.group_sizes = np.zeros(cap, np.int32) if want_stats else None
        self.nodes_added = np.zeros(cap, np.int32) if want_stats else None
        self.collision_checks = np.zeros(cap, np.int64) if want_stats else None
        self.out = PlanOut()
        o = self.out
        o.stats_cap = cap if want_stats else 0
        o.path = ptr(self.path, C.c_int32)
        o.label = ptr(self.label, C.c_uint8)
        o.tree_cost = ptr(self.tree_cost, C.c_double)
        o.parent = ptr(self.parent, C.c_int32)
        o.iteration_added = ptr(self.iteration_added, C.c_int64)
        o.group_sizes = ptr(self.group_sizes, C.c_int32)
        o.nodes_added = ptr(self.nodes_added, C.c_int32)
        o.collision_checks = ptr(self.collision_checks, C.c_int64)

    def result(self) -> "PlanResultPy":
        o = self.out
        t = o.tree_size
        s = o.num_stats
        return PlanResultPy(
            status=o.status,
            cost=o.cost,
            iterations=o.iterations,
            total_collision_checks=o.total_collision_checks,
            path_indices=self.path[: o.path_len].copy(),
            label=None if self.label is None else self.label[:t].copy(),
            tree_cost=None if self.tree_cost is None else self.tree_cost[:t].copy(),
            parent=None if self.parent is None else self.parent[:t].copy(),
            iteration_added=None if self.iteration_added is None else self.iteration_added[:t].copy(),
            group_sizes=None if self.group_sizes is None else self.group_sizes[:s].copy(),
            nodes_added=None if self.nodes_added is None else self.nodes_added[:s].copy(),
            collision_checks=None if self.collision_checks is None else self.collision_checks[:s].copy(),
        )


class PlanResultPy:
    """PlanResult (planner.hpp:43-51) as numpy arrays."""

    __slots__ = (
        "status", "cost", "iterations", "total_collision_checks", "path_indices", "label",
        "tree_cost", "parent", "iteration_added", "group_sizes", "nodes_added",
        "collision_checks",
    )

    def __init__(self, **kw):
        for k in self.__slots__:
            setattr(self, k, kw.get(k))

    def __repr__(self):
        return (f"PlanResult(status={self.status}, cost={self.cost!r}, iterations={self.iterations}, "
                f"checks={self.total_collision_checks}, path_len={len(self.path_indices)})")


def same_tree(a: PlanResultPy, b: PlanResultPy) -> bool:
    """Bitwise tree equality, the reference's `same_tree`
    (tests/support/oracles.cpp:329-341): status, path, parent, label, the cost
    array compared as raw bits, and the result cost as raw bits."""
    if a.status != b.status:
        return False
    if not np.array_equal(a.path_indices, b.path_indices):
        return False
    if not np.array_equal(a.parent, b.parent) or not np.array_equal(a.label, b.label):
        return False
    if a.tree_cost.shape != b.tree_cost.shape:
        return False
    if a.tree_cost.view(np.uint64).tolist() != b.tree_cost.view(np.uint64).tolist():
        return False
    return np.float64(a.cost).view(np.uint64) == np.float64(b.cost).view(np.uint64)


def full_parity(a: PlanResultPy, b: PlanResultPy) -> list[str]:
    """same_tree plus every other PlanResult field (BASELINE.md §4 parity gate:
    iterations, total_collision_checks, iteration_added and per-pass stats).
    Returns the list of mismatching fields (empty = identical)."""
    bad = []
    if not same_tree(a, b):
        bad.append("same_tree")
    if a.iterations != b.iterations:
        bad.append("iterations")
    if a.total_collision_checks != b.total_collision_checks:
        bad.append("total_collision_checks")
    for f in ("iteration_added", "group_sizes", "nodes_added", "collision_checks"):
        x, y = getattr(a, f), getattr(b, f)
        if x is None or y is None:
            continue
        if not np.array_equal(x, y):
            bad.append(f)
    return bad


class Scenario(C.Structure):
    """gmt_scenario: ScenarioConfig + PlanningSetup (simulator.hpp:14-36)."""
    _fields_ = [
        ("scene", Scene),
        ("init", _dp),
        ("n", C.c_int32),
        ("trials", C.c_int32),
        ("lambda_", C.c_double),
        ("eta", C.c_double),
        ("radius_override", C.c_double),
        ("collapse_rate", C.c_double),
        ("spawn_box_size", C.c_double),
        ("disturbance_sigma", C.c_double),
        ("replan_latency", C.c_double),
        ("control_dt", C.c_double),
        ("robot_speed", C.c_double),
        ("time_limit", C.c_double),
        ("seed", C.c_uint64),
    ]


class TrialOutcome(C.Structure):
    """gmt_trial_outcome (simulator.hpp:40-51)."""
    _fields_ = [
        ("result", C.c_int32),
        ("replans", C.c_int32),
        ("spawned", C.c_int32),
        ("noise_outliers", C.c_int32),
        ("time", C.c_double),
        ("path_len", C.c_int64),
    ]


TRIAL_REACHED_GOAL, TRIAL_COLLIDED, TRIAL_TIMED_OUT = 0, 1, 2

