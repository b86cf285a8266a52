"""Problem description (gmt-problem/1) on the host side.

`ProblemSpec` mirrors `gmt::ProblemFile` (problem.hpp:17-29) for the
Euclidean model, `load_problem`/`parse_problem` mirror the reference's strict
JSON loader (problem.cpp:102-231: unknown keys rejected at every level,
errors name the offending field path, init must be free), and the synthetic
scene generators define the BASELINE workloads that have no reference scene
file: the 3D forest (C2) and the batched query sets.
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field

import numpy as np

from . import abi
from .errors import InvalidInputError

# 12D quadrotor units: the unit workspace cube is 10 m, so g = 0.981 per s^2.
QUAD_G = 0.981
QUAD_RADIUS = 3.5

SCHEMA = "gmt-problem/1"
MASK64 = (1 << 64) - 1


# ---- PCG32 / splitmix64 (rng.hpp:11-75), host-side scene generation only ----
class Pcg32:
    """PCG-XSH-RR 32 exactly as rng.hpp:11-33 (used to draw synthetic scenes)."""

    def __init__(self, seed: int, seq: int = 0):
        self.state = 0
        self.inc = ((seq << 1) | 1) & MASK64
        self.next_u32()
        self.state = (self.state + seed) & MASK64
        self.next_u32()

    def next_u32(self) -> int:
        old = self.state
        self.state = (old * 6364136223846793005 + self.inc) & MASK64
        xorshifted = (((old >> 18) ^ old) >> 27) & 0xFFFFFFFF
        rot = old >> 59
        return ((xorshifted >> rot) | (xorshifted << ((32 - rot) & 31))) & 0xFFFFFFFF

    def next_double(self) -> float:
        return self.next_u32() * 2.0 ** -32


def mix64(x: int, b: int | None = None) -> int:
    """splitmix64 (rng.hpp:68-75); mix64(a, b) = mix64(mix64(a) ^ b)."""
    if b is not None:
        return mix64(mix64(x) ^ b)
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
    return x ^ (x >> 31)


@dataclass
class ProblemSpec:
    dim: int
    box_lo: np.ndarray  # [B, dim]
    box_hi: np.ndarray  # [B, dim]
    goal_lo: np.ndarray  # [dim]
    goal_hi: np.ndarray  # [dim]
    init: np.ndarray  # [dim]
    n: int
    lam: float = 1.0
    eta: float = 0.0
    radius_override: float | None = None
    sampling_kind: int = abi.SAMPLE_HALTON
    start_index: int = 1
    seed: int = 0
    notes: str = ""
    steering: int = abi.STEER_EUCLIDEAN
    di_vmax: float = 0.5
    di_weight: float = 1.0
    di_segments: int = 8
    quad_g: float = QUAD_G
    quad_vmax: float = 0.5
    quad_amax: float = 0.5
    quad_ymax: float = math.pi
    quad_wmax: float = 1.0
    quad_weight: float = 0.1
    init_heading: float | None = None  # Dubins problems (State::heading)
    dubins_rho: float = 0.1
    dubins_step: float = 0.0
    dubins_planar: bool = False
    quad_segments: int = 8
    _keep: list = field(default_factory=list, repr=False)

    def di_params(self) -> abi.DiParams:
        p = abi.DiParams()
        p.vmax, p.weight, p.segments, p.reserved = self.di_vmax, self.di_weight, self.di_segments, 0
        return p

    def quad_params(self) -> abi.QuadParams:
        p = abi.QuadParams()
        p.g, p.vmax, p.amax, p.ymax, p.wmax, p.weight = (
            self.quad_g, self.quad_vmax, self.quad_amax, self.quad_ymax, self.quad_wmax,
            self.quad_weight)
        p.segments, p.reserved = self.quad_segments, 0
        return p

    @property
    def num_boxes(self) -> int:
        return int(self.box_lo.shape[0])

    def scene(self) -> abi.Scene:
        """Flat gmt_scene view (keeps the arrays alive on self)."""
        lo = abi.f64(self.box_lo.reshape(-1)) if self.num_boxes else np.zeros(1)
        hi = abi.f64(self.box_hi.reshape(-1)) if self.num_boxes else np.zeros(1)
        gl, gh = abi.f64(self.goal_lo), abi.f64(self.goal_hi)
        self._keep = [lo, hi, gl, gh]
        s = abi.Scene()
        s.dim = self.dim
        s.num_boxes = self.num_boxes
        s.box_lo = abi.ptr(lo, abi.C.c_double)
        s.box_hi = abi.ptr(hi, abi.C.c_double)
        s.goal_lo = abi.ptr(gl, abi.C.c_double)
        s.goal_hi = abi.ptr(gh, abi.C.c_double)
        return s

    def source(self) -> abi.SampleSource:
        s = abi.SampleSource()
        s.kind = self.sampling_kind
        s.with_heading = 1 if self.steering == abi.STEER_DUBINS_AIRPLANE else 0  # problem.cpp:197
        s.start_index = self.start_index
        s.seed = self.seed
        return s

    def flat(self) -> abi.Problem:
        p = abi.Problem()
        p.scene = self.scene()
        init = abi.f64(self.init)
        self._keep.append(init)
        p.init = abi.ptr(init, abi.C.c_double)
        p.init_has_heading = 0 if self.init_heading is None else 1
        p.init_heading = 0.0 if self.init_heading is None else float(self.init_heading)
        p.n = self.n
        p.lambda_ = self.lam
        p.eta = self.eta
        p.radius_override = self.radius_override if self.radius_override else 0.0
        p.sampling = self.source()
        p.steering = self.steering
        p.reserved = 0
        p.di = self.di_params()
        p.quad = self.quad_params()
        p.dubins = self.dubins_params()
        return p

    def dubins_params(self) -> abi.DubinsParams:
        d = abi.DubinsParams()
        d.rho, d.discretization_step = self.dubins_rho, self.dubins_step
        d.planar_cost_only, d.reserved = int(self.dubins_planar), 0
        return d

    def with_n(self, n: int) -> "ProblemSpec":
        q = ProblemSpec(**{k: getattr(self, k) for k in self.__dataclass_fields__ if k != "_keep"})
        q.n = n
        return q

    def point_free(self, p) -> bool:
        """point_free (space.cpp:47-54)."""
        p = np.asarray(p, np.float64)
        if np.any(p < 0.0) or np.any(p > 1.0):
            return False
        for b in range(self.num_boxes):
            if np.all(p >= self.box_lo[b]) and np.all(p <= self.box_hi[b]):
                return False
        return True

    def to_json(self) -> str:
        """problem_json (problem.cpp:233-272), Euclidean model."""
        doc = {
            "schema": SCHEMA,
            "dimension": self.dim,
            "steering": {"model": "euclidean"},
            "obstacles": [{"lo": self.box_lo[b].tolist(), "hi": self.box_hi[b].tolist()}
                          for b in range(self.num_boxes)],
            "init": {"coords": self.init.tolist()},
            "goal": {"lo": self.goal_lo.tolist(), "hi": self.goal_hi.tolist()},
            "n": self.n,
            "lambda": self.lam,
            "eta": self.eta,
        }
        if self.radius_override:
            doc["radius_override"] = self.radius_override
        if self.sampling_kind == abi.SAMPLE_HALTON:
            doc["sampling"] = {"kind": "halton", "start_index": self.start_index}
        else:
            doc["sampling"] = {"kind": "uniform", "seed": self.seed}
        if self.notes:
            doc["notes"] = self.notes
        return json.dumps(doc, indent=2) + "\n"


# ---- strict loader (problem.cpp:102-231) ----------------------------------
def _fail(path: str, what: str):
    raise InvalidInputError(f"{path}: {what}")


def _reject_unknown(obj: dict, path: str, allowed):
    for k in obj:
        if k not in allowed:
            _fail(k if not path else f"{path}.{k}", "unknown field")


def _member(obj: dict, path: str, key: str):
    if key not in obj:
        _fail(key if not path else f"{path}.{key}", "required field is missing")
    return obj[key]


def _is_num(v) -> bool:
    return isinstance(v, (int, float)) and not isinstance(v, bool)


def _as_double(v, path):
    if not _is_num(v):
        _fail(path, "expected a number")
    return float(v)


def _as_int(v, path):
    if not isinstance(v, int) or isinstance(v, bool):
        _fail(path, "expected an integer")
    return v


def _as_vector(v, path, dim):
    if not isinstance(v, list):
        _fail(path, "expected an array of numbers")
    if len(v) != dim:
        _fail(path, f"expected {dim} coordinates, got {len(v)}")
    return np.array([_as_double(x, f"{path}[{k}]") for k, x in enumerate(v)], np.float64)


def _parse_box(v, path, dim):
    if not isinstance(v, dict):
        _fail(path, "expected an object with lo and hi")
    _reject_unknown(v, path, ("lo", "hi"))
    lo = _as_vector(_member(v, path, "lo"), path + ".lo", dim)
    hi = _as_vector(_member(v, path, "hi"), path + ".hi", dim)
    for k in range(dim):
        if lo[k] > hi[k]:
            _fail(path, f"lo exceeds hi on axis {k}")
    return lo, hi


def parse_problem(text: str) -> ProblemSpec:
    """parse_problem (problem.cpp:102-223): euclidean and dubins_airplane
    steering (the latter with its rho / discretization_step /
    planar_cost_only fields and a required init heading)."""
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise InvalidInputError(f"invalid JSON: {e}") from None
    if not isinstance(doc, dict):
        raise InvalidInputError("top level: expected a JSON object")
    _reject_unknown(doc, "", ("schema", "dimension", "steering", "obstacles", "init", "goal", "n",
                              "lambda", "eta", "radius_override", "sampling", "notes"))
    schema = _member(doc, "", "schema")
    if not isinstance(schema, str):
        _fail("schema", "expected a string")
    if schema != SCHEMA:
        _fail("schema", f'expected "{SCHEMA}"')
    dim = _as_int(_member(doc, "", "dimension"), "dimension")
    if dim < 1:
        _fail("dimension", "must be at least 1")
    steering = _member(doc, "", "steering")
    dubins = {}
    if not isinstance(steering, dict):
        _fail("steering", "expected an object")
    _reject_unknown(steering, "steering", ("model", "rho", "discretization_step", "planar_cost_only"))
    model = _member(steering, "steering", "model")
    if not isinstance(model, str):
        _fail("steering.model", "expected a string")
    if model == "euclidean":
        for key in ("rho", "discretization_step", "planar_cost_only"):
            if key in steering:
                _fail(f"steering.{key}", "only the dubins_airplane model uses this field")
    elif model == "dubins_airplane":  # problem.cpp:132-151
        if dim not in (2, 3):
            _fail("dimension", "dubins_airplane needs dimension 2 or 3")
        if "rho" in steering:
            rho = _as_double(steering["rho"], "steering.rho")
            if not rho > 0.0:
                _fail("steering.rho", "must be positive")
            dubins["rho"] = rho
        if "discretization_step" in steering:
            st = _as_double(steering["discretization_step"], "steering.discretization_step")
            if st < 0.0:
                _fail("steering.discretization_step", "must be non-negative")
            dubins["step"] = st
        if "planar_cost_only" in steering:
            if not isinstance(steering["planar_cost_only"], bool):
                _fail("steering.planar_cost_only", "expected a boolean")
            dubins["planar"] = steering["planar_cost_only"]
    else:
        _fail("steering.model", 'expected "euclidean" or "dubins_airplane"')
    obstacles = _member(doc, "", "obstacles")
    if not isinstance(obstacles, list):
        _fail("obstacles", "expected an array of boxes")
    los, his = [], []
    for k, b in enumerate(obstacles):
        lo, hi = _parse_box(b, f"obstacles[{k}]", dim)
        los.append(lo)
        his.append(hi)
    box_lo = np.array(los, np.float64).reshape(-1, dim)
    box_hi = np.array(his, np.float64).reshape(-1, dim)
    init = _member(doc, "", "init")
    if not isinstance(init, dict):
        _fail("init", "expected an object with coords")
    _reject_unknown(init, "init", ("coords", "heading"))
    init_c = _as_vector(_member(init, "init", "coords"), "init.coords", dim)
    is_dubins = steering.get("model") == "dubins_airplane"
    init_heading = None
    if "heading" in init:  # problem.cpp:165-173
        if not is_dubins:
            _fail("init.heading", "only the dubins_airplane model uses a heading")
        init_heading = _as_double(init["heading"], "init.heading")
    elif is_dubins:
        _fail("init.heading", "required field is missing")
    goal_lo, goal_hi = _parse_box(_member(doc, "", "goal"), "goal", dim)
    n = _as_int(_member(doc, "", "n"), "n")
    if n < 1:
        _fail("n", "must be at least 1")
    spec = ProblemSpec(dim=dim, box_lo=box_lo, box_hi=box_hi, goal_lo=goal_lo, goal_hi=goal_hi,
                       init=init_c, n=n)
    if is_dubins:
        spec.steering = abi.STEER_DUBINS_AIRPLANE
        spec.init_heading = init_heading
        spec.dubins_rho = dubins.get("rho", 0.1)
        spec.dubins_step = dubins.get("step", 0.0)
        spec.dubins_planar = bool(dubins.get("planar", False))
    if not spec.point_free(init_c):
        _fail("init", "start state is not in free space")
    if "lambda" in doc:
        lam = _as_double(doc["lambda"], "lambda")
        if not lam > 0.0 or lam > 1.0:
            _fail("lambda", "must be in (0, 1]")
        spec.lam = lam
    if "eta" in doc:
        eta = _as_double(doc["eta"], "eta")
        if eta < 0.0:
            _fail("eta", "must be non-negative")
        spec.eta = eta
    if "radius_override" in doc:
        r = _as_double(doc["radius_override"], "radius_override")
        if not r > 0.0:
            _fail("radius_override", "must be positive")
        spec.radius_override = r
    if "sampling" in doc:
        s = doc["sampling"]
        if not isinstance(s, dict):
            _fail("sampling", "expected an object")
        _reject_unknown(s, "sampling", ("kind", "start_index", "seed"))
        kind = _member(s, "sampling", "kind")
        if not isinstance(kind, str):
            _fail("sampling.kind", "expected a string")
        if kind == "halton":
            spec.sampling_kind = abi.SAMPLE_HALTON
            if "seed" in s:
                _fail("sampling.seed", "only uniform sampling takes a seed")
            if "start_index" in s:
                v = s["start_index"]
                if not isinstance(v, int) or isinstance(v, bool) or v < 0:
                    _fail("sampling.start_index", "expected a non-negative integer")
                if v == 0:
                    _fail("sampling.start_index", "must be at least 1")
                spec.start_index = v
        elif kind == "uniform":
            spec.sampling_kind = abi.SAMPLE_UNIFORM
            if "start_index" in s:
                _fail("sampling.start_index", "only halton sampling takes a start index")
            if "seed" in s:
                v = s["seed"]
                if not isinstance(v, int) or isinstance(v, bool) or v < 0:
                    _fail("sampling.seed", "expected a non-negative integer")
                spec.seed = v
        else:
            _fail("sampling.kind", 'expected "halton" or "uniform"')
    if "notes" in doc:
        if not isinstance(doc["notes"], str):
            _fail("notes", "expected a string")
        spec.notes = doc["notes"]
    return spec


def load_problem(path: str) -> ProblemSpec:
    """load_problem (problem.cpp:225-231)."""
    try:
        with open(path, "rb") as f:
            text = f.read().decode()
    except OSError:
        raise InvalidInputError(f"{path}: cannot open file") from None
    return parse_problem(text)


# ---- synthetic BASELINE scenes ---------------------------
def forest_3d(seed: int = 3, n: int = 4000, pillars: int = 60) -> ProblemSpec:
    """C2 "3D forest": `pillars` vertical boxes drawn from Pcg32(seed):
    centre U[0.1,0.9]^2, square footprint half-width U[0.02,0.05], z from 0 to
    a height U[0.5,1].  Init (0.03,0.03,0.5); goal [0.92,0.98]^2 x [0.4,0.6];
    Halton samples; formula radius."""
    rng = Pcg32(seed)
    lo, hi = [], []
    for _ in range(pillars):
        cx = 0.1 + 0.8 * rng.next_double()
        cy = 0.1 + 0.8 * rng.next_double()
        hw = 0.02 + 0.03 * rng.next_double()
        h = 0.5 + 0.5 * rng.next_double()
        lo.append([cx - hw, cy - hw, 0.0])
        hi.append([cx + hw, cy + hw, h])
    spec = ProblemSpec(dim=3, box_lo=np.array(lo), box_hi=np.array(hi),
                       goal_lo=np.array([0.92, 0.92, 0.4]), goal_hi=np.array([0.98, 0.98, 0.6]),
                       init=np.array([0.03, 0.03, 0.5]), n=n,
                       notes=f"Synthetic 3D forest: {pillars} pillars from Pcg32({seed}).")
    if not spec.point_free(spec.init):
        raise InvalidInputError("forest init collides")
    return spec


def random_forest_query(master: int, q: int, n: int = 4000, pillars: int = 60) -> ProblemSpec:
    """Batched query q (SURVEY.md §8(d) C5 construction, Euclidean 3D): its own
    forest, start and goal drawn from Pcg32(mix64(master, q)).  Start in the
    low corner region, goal box in the opposite corner region."""
    rng = Pcg32(mix64(master, q))
    lo, hi = [], []
    for _ in range(pillars):
        cx = 0.1 + 0.8 * rng.next_double()
        cy = 0.1 + 0.8 * rng.next_double()
        hw = 0.02 + 0.03 * rng.next_double()
        h = 0.5 + 0.5 * rng.next_double()
        lo.append([cx - hw, cy - hw, 0.0])
        hi.append([cx + hw, cy + hw, h])
    box_lo, box_hi = np.array(lo), np.array(hi)
    spec = None
    for _ in range(100):
        init = np.array([0.02 + 0.06 * rng.next_double(), 0.02 + 0.06 * rng.next_double(),
                         0.2 + 0.6 * rng.next_double()])
        gc = np.array([0.90 + 0.05 * rng.next_double(), 0.90 + 0.05 * rng.next_double(),
                       0.3 + 0.4 * rng.next_double()])
        spec = ProblemSpec(dim=3, box_lo=box_lo, box_hi=box_hi, goal_lo=gc - 0.04,
                           goal_hi=np.minimum(gc + 0.04, 1.0), init=init, n=n)
        if spec.point_free(init):
            return spec
    raise InvalidInputError("could not draw a free start")


def extrude(spec: ProblemSpec, dim: int, n: int | None = None) -> ProblemSpec:
    """Lift a scene to `dim` dimensions by extruding every box through the
    extra axes (the construction of rectangles_6d.json and the SURVEY's 12D
    stand-in, §6 C4).  Init/goal take 0.5 / [0.2,0.8] on new axes."""
    extra = dim - spec.dim
    box_lo = np.concatenate([spec.box_lo, np.zeros((spec.num_boxes, extra))], axis=1)
    box_hi = np.concatenate([spec.box_hi, np.ones((spec.num_boxes, extra))], axis=1)
    return ProblemSpec(dim=dim, box_lo=box_lo, box_hi=box_hi,
                       goal_lo=np.concatenate([spec.goal_lo, np.full(extra, 0.2)]),
                       goal_hi=np.concatenate([spec.goal_hi, np.full(extra, 0.8)]),
                       init=np.concatenate([spec.init, np.full(extra, 0.5)]),
                       n=spec.n if n is None else n, lam=spec.lam, eta=spec.eta,
                       radius_override=spec.radius_override)


def random_problem_2d(rng: Pcg32, dim: int = 2, with_obstacles: bool = True, n_min: int = 120,
                      n_max: int = 350):
    """make_random_problem (tests/support/oracles.cpp:258-327), Euclidean
    branch, draw for draw: 2-6 boxes, goal box, free init not in goal,
    uniform samples seeded mix64(u32, u32), n in [n_min, n_max].  Returns
    the spec; sampling failures are retried by the caller's loop like the
    reference (which catches runtime_error and redraws)."""
    for _ in range(200):
        lo, hi = [], []
        if with_obstacles:
            count = 2 + rng.next_u32() % 5
            for _b in range(count):
                l, h = [], []
                for _k in range(dim):
                    a = rng.next_double() * 0.85
                    size = 0.05 + 0.20 * rng.next_double()
                    l.append(a)
                    h.append(min(a + size, 1.0))
                lo.append(l)
                hi.append(h)
        gl, gh = [], []
        for _k in range(dim):
            c = 0.15 + 0.7 * rng.next_double()
            half = 0.04 + 0.04 * rng.next_double()
            gl.append(max(c - half, 0.0))
            gh.append(min(c + half, 1.0))
        spec = ProblemSpec(dim=dim, box_lo=np.array(lo, np.float64).reshape(-1, dim),
                           box_hi=np.array(hi, np.float64).reshape(-1, dim),
                           goal_lo=np.array(gl), goal_hi=np.array(gh), init=np.zeros(dim), n=1)
        found = False
        for _t in range(400):
            p = np.array([rng.next_double() for _k in range(dim)])
            in_goal = bool(np.all(p >= spec.goal_lo) and np.all(p <= spec.goal_hi))
            if spec.point_free(p) and not in_goal:
                spec.init = p
                found = True
                break
        if not found:
            continue
        spec.sampling_kind = abi.SAMPLE_UNIFORM
        # mix64(rng.next_u32(), rng.next_u32()) (oracles.cpp:303): GCC on
        # x86-64 evaluates the arguments right to left, so the FIRST draw is
        # the second argument.  Pinned by tests/test_oracle.py.
        first = rng.next_u32()
        second = rng.next_u32()
        spec.seed = mix64(second, first)
        spec.n = n_min + rng.next_u32() % (n_max - n_min + 1)
        return spec
    raise RuntimeError("random problem generation kept hitting infeasible draws")


def di_forest(seed: int = 3, n: int = 4000, pillars: int = 60, radius: float = 1.6,
              vmax: float = 0.5) -> ProblemSpec:
    """C3 "6D double integrator in a 3D obstacle field":
    the C2 forest's pillars extruded over the full normalised velocity range,
    state [p, s] with v = vmax (2s - 1); start at rest in the low corner,
    goal = a position box with speeds below vmax/2 on every axis; Halton
    samples; the connection radius is a cost threshold (radius_override)."""
    base = forest_3d(seed, n, pillars)
    box_lo = np.concatenate([base.box_lo, np.zeros((base.num_boxes, 3))], axis=1)
    box_hi = np.concatenate([base.box_hi, np.ones((base.num_boxes, 3))], axis=1)
    spec = ProblemSpec(dim=6, box_lo=box_lo, box_hi=box_hi,
                       goal_lo=np.array([0.90, 0.90, 0.35, 0.25, 0.25, 0.25]),
                       goal_hi=np.array([0.98, 0.98, 0.65, 0.75, 0.75, 0.75]),
                       init=np.array([0.03, 0.03, 0.5, 0.5, 0.5, 0.5]), n=n,
                       radius_override=radius, steering=abi.STEER_DOUBLE_INTEGRATOR,
                       di_vmax=vmax, notes=f"6D double integrator, forest Pcg32({seed}).")
    return spec


def random_di_query(master: int, q: int, n: int = 4000, pillars: int = 60,
                    radius: float = 1.6) -> ProblemSpec:
    """C5 batched 6D double-integrator query q: its own forest, start and
    goal from Pcg32(mix64(master, q)) (random_forest_query extruded)."""
    base = random_forest_query(master, q, n=n, pillars=pillars)
    box_lo = np.concatenate([base.box_lo, np.zeros((base.num_boxes, 3))], axis=1)
    box_hi = np.concatenate([base.box_hi, np.ones((base.num_boxes, 3))], axis=1)
    return ProblemSpec(dim=6, box_lo=box_lo, box_hi=box_hi,
                       goal_lo=np.concatenate([base.goal_lo, np.full(3, 0.25)]),
                       goal_hi=np.concatenate([base.goal_hi, np.full(3, 0.75)]),
                       init=np.concatenate([base.init, np.full(3, 0.5)]), n=n,
                       radius_override=radius, steering=abi.STEER_DOUBLE_INTEGRATOR)


def quad_scene(seed: int = 5, n: int = 8000, pillars: int = 90, beams: int = 40,
               radius: float = QUAD_RADIUS, position_goal: bool = False) -> ProblemSpec:
    """C4 "12D linearised quadrotor, complex box scene":
    a 3D scene of `pillars` forest pillars plus `beams` horizontal beams
    (Pcg32(seed)), extruded over the full range of the nine non-position
    coordinates; start hovering at rest in the low corner, goal = a position
    box in the far corner with |v| < 0.8 vmax, |roll|, |pitch| < 0.8 amax,
    any yaw, |rates| < 0.8 wmax (about 15 goal samples at n = 8000);
    Halton samples; the connection radius is a cost threshold.
    position_goal: the goal constrains the position only (small-n tests)."""
    rng = Pcg32(seed)
    lo, hi = [], []
    for _ in range(pillars):
        cx = 0.1 + 0.8 * rng.next_double()
        cy = 0.1 + 0.8 * rng.next_double()
        hw = 0.02 + 0.03 * rng.next_double()
        h = 0.5 + 0.5 * rng.next_double()
        lo.append([cx - hw, cy - hw, 0.0])
        hi.append([cx + hw, cy + hw, h])
    for _ in range(beams):  # axis-aligned beams at random heights
        ax = rng.next_u32() % 2
        c = 0.1 + 0.8 * rng.next_double()
        z = 0.1 + 0.8 * rng.next_double()
        a = 0.8 * rng.next_double()
        ln = 0.1 + 0.3 * rng.next_double()
        hw = 0.01 + 0.02 * rng.next_double()
        if ax == 0:
            lo.append([a, c - hw, z - hw])
            hi.append([min(a + ln, 1.0), c + hw, z + hw])
        else:
            lo.append([c - hw, a, z - hw])
            hi.append([c + hw, min(a + ln, 1.0), z + hw])
    B = len(lo)
    box_lo = np.concatenate([np.array(lo).reshape(B, 3), np.zeros((B, 9))], axis=1)
    box_hi = np.concatenate([np.array(hi).reshape(B, 3), np.ones((B, 9))], axis=1)
    init = np.array([0.03, 0.03, 0.5] + [0.5] * 9)
    glo = np.array([0.85, 0.85, 0.25] + [0.1] * 5 + [0.0] + [0.1] * 3)
    ghi = np.array([1.0, 1.0, 0.75] + [0.9] * 5 + [1.0] + [0.9] * 3)
    if position_goal:
        glo[3:], ghi[3:] = 0.0, 1.0
    spec = ProblemSpec(dim=12, box_lo=box_lo, box_hi=box_hi, goal_lo=glo, goal_hi=ghi, init=init,
                       n=n, radius_override=radius, steering=abi.STEER_QUADROTOR,
                       notes=f"12D quadrotor, {pillars} pillars + {beams} beams, Pcg32({seed}).")
    if not spec.point_free(init):
        raise InvalidInputError("quadrotor init collides")
    return spec


def halton_pool_size(specs) -> int:
    """Halton points a shared sample pool needs for `specs` (SURVEY.md
    §8(e)): n over the free-volume estimate (boxes clipped to the unit cube,
    overlaps counted twice), +5 % + 256 -- the device pool's own sizing
    (csrc/pool.cu: pool_need)."""
    need = 0
    for s in specs:
        lo = np.clip(s.box_lo, 0.0, 1.0)
        hi = np.clip(s.box_hi, 0.0, 1.0)
        blocked = float(np.clip(hi - lo, 0.0, None).prod(axis=1).sum()) if s.num_boxes else 0.0
        need = max(need, int(math.ceil(min(4.0 * s.n, s.n / max(0.05, 1.0 - blocked) * 1.05) + 256)))
    return need


def connection_radius_py(dim: int, n: int, eta: float = 0.0, mu: float = 1.0) -> float:
    """Python float restatement of graph.cpp:19-32 (for quick checks only;
    the product computes it in C++ with the same libm calls)."""
    inv_d = 1.0 / dim
    zeta = math.pi ** (0.5 * dim) / math.gamma(0.5 * dim + 1.0)
    return (4.0 * (1.0 + eta) ** inv_d * inv_d ** inv_d * (mu / zeta) ** inv_d
            * (math.log(n) / n) ** inv_d)


@dataclass
class Scenario:
    """ScenarioConfig (simulator.hpp:25-36) over a planning setup given as a
    ProblemSpec (obstacles at t = 0, goal, init, n, lambda, eta, radius)."""
    spec: ProblemSpec
    collapse_rate: float = 0.0
    spawn_box_size: float = 0.08
    disturbance_sigma: float = 0.0
    replan_latency: float = 0.1
    control_dt: float = 0.05
    robot_speed: float = 0.1
    time_limit: float = 30.0
    trials: int = 50
    seed: int = 0
    _keep: list = field(default_factory=list, repr=False)

    def flat(self) -> abi.Scenario:
        s = abi.Scenario()
        s.scene = self.spec.scene()
        init = abi.f64(self.spec.init)
        self._keep = [init, self.spec._keep]
        s.init = abi.ptr(init, abi.C.c_double)
        s.n = self.spec.n
        s.trials = self.trials
        s.lambda_ = self.spec.lam
        s.eta = self.spec.eta
        s.radius_override = self.spec.radius_override or 0.0
        for f in ("collapse_rate", "spawn_box_size", "disturbance_sigma", "replan_latency",
                  "control_dt", "robot_speed", "time_limit"):
            setattr(s, f, getattr(self, f))
        s.seed = self.seed
        return s

