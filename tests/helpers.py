"""Shared test helpers: build reference-side problem instances with the
oracle so GPU results can be compared on identical samples and graphs."""
from __future__ import annotations

import json
import os

import numpy as np

from paper_1705_02403_b200 import problem as P
from paper_1705_02403_b200.graph import Graph

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
_SCENES = None


def golden(name: str):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def scene(name: str, n: int | None = None) -> P.ProblemSpec:
    """A bundled reference scene (proj/scenes/<name>.json), from the fixture
    the reference's own parser produced (tests/golden/make_golden.py)."""
    global _SCENES
    if _SCENES is None:
        _SCENES = golden("scenes.json")
    e = _SCENES[name]
    d = e["dim"]
    spec = P.ProblemSpec(dim=d, box_lo=np.array(e["box_lo"], np.float64).reshape(-1, d),
                         box_hi=np.array(e["box_hi"], np.float64).reshape(-1, d),
                         goal_lo=np.array(e["goal_lo"]), goal_hi=np.array(e["goal_hi"]),
                         init=np.array(e["init"]), n=e["n"], lam=e["lambda"], eta=e["eta"],
                         radius_override=e["radius_override"], sampling_kind=e["sampling_kind"],
                         start_index=e["start_index"], seed=e["seed"])
    return spec if n is None else spec.with_n(n)


SCENE_NAMES = ["rectangles_2d", "rectangles_3d", "rectangles_6d", "maze_3d", "cave_sim"]


def oracle_instance(lib, spec, radius: float | None = None):
    """sample_free -> append_init -> radius -> graph with the given oracle
    library (port or ref).  Returns dict(coords, goal_idx, init, radius, graph)."""
    coords, gidx = lib.sample_free(spec)
    coords, gidx, ii = lib.append_init(coords, gidx, spec.init, spec.goal_lo, spec.goal_hi)
    if radius is None:
        radius = spec.radius_override or lib.connection_radius(spec.dim, spec.n, spec.eta)
    ptr, col, cost = lib.build_neighbor_graph(coords, radius)
    g = Graph(coords.shape[0], radius, ptr, col, cost, dim=spec.dim)
    return dict(coords=coords, goal_idx=gidx, init=ii, radius=radius, graph=g)


def random_ref_problem(ref, rng, **kw):
    """The reference's make_random_problem (oracles.cpp:258-327) + its graph."""
    p = ref.random_problem(rng, **kw)
    ptr, col, cost = ref.build_neighbor_graph(p["coords"], p["radius"])
    p["graph"] = Graph(p["coords"].shape[0], p["radius"], ptr, col, cost, dim=p["spec"].dim)
    return p


def bits(a: np.ndarray) -> bytes:
    return np.ascontiguousarray(a).view(np.uint64).tobytes()


def forest_dubins(n: int = 600) -> P.ProblemSpec:
    """proj/scenes/forest_dubins.json (8 square pillars, rho = 0.08, pinned
    radius 0.2, Halton samples with headings)."""
    from paper_1705_02403_b200 import abi
    lo = [[0.21, 0.21], [0.21, 0.56], [0.26, 0.81], [0.46, 0.36], [0.51, 0.71], [0.61, 0.11],
          [0.71, 0.51], [0.81, 0.76]]
    box_lo = np.array(lo)
    return P.ProblemSpec(dim=2, box_lo=box_lo, box_hi=box_lo + 0.08, goal_lo=np.array([0.88, 0.88]),
                         goal_hi=np.array([0.98, 0.98]), init=np.array([0.05, 0.05]), n=n,
                         radius_override=0.2, steering=abi.STEER_DUBINS_AIRPLANE, init_heading=0.0,
                         dubins_rho=0.08)
