"""CPU tests of the oracle itself (no GPU): the C restatement
(oracle/gmt_oracle.c) is pinned against the committed golden vectors of the
unmodified reference, and -- where the compiled reference is present --
against the reference directly, bit for bit."""
import hashlib

import numpy as np
import pytest

from paper_1705_02403_b200 import abi, problem as P
from paper_1705_02403_b200.errors import (GoalBlockedError, InfeasibleSamplingError,
                                          InvalidInputError)
from paper_1705_02403_b200.graph import Graph
from helpers import SCENE_NAMES, bits, golden, oracle_instance, scene


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def hexf(x):
    return np.float64(x).tobytes().hex()


def test_halton_prime_kats(port):
    k = golden("kats.json")
    for i, b, h in k["halton"]:
        assert hexf(port.halton(i, b)) == h
    for kk, p in k["nth_prime"]:
        assert port.nth_prime(kk) == p
    # test_sampling.cpp:29-47
    assert port.halton(1, 2) == 0.5 and port.halton(3, 2) == 0.75
    assert abs(port.halton(5, 3) - 7.0 / 9.0) < 1e-15
    with pytest.raises(InvalidInputError):
        port.halton(0, 2)
    with pytest.raises(InvalidInputError):
        port.halton(1, 4)
    with pytest.raises(InvalidInputError):
        port.nth_prime(0)


def test_radius_kats(port):
    k = golden("kats.json")
    for d, n, eta, mu, h in k["radius"]:
        assert hexf(port.connection_radius(d, n, eta, mu)) == h
    for d, h in k["unit_ball"]:
        assert hexf(port.unit_ball_volume(d)) == h
    assert abs(port.connection_radius(2, 1000) - 0.13263) < 1e-4 * 0.13263  # test_graph.cpp:44-49
    with pytest.raises(InvalidInputError):
        port.connection_radius(2, 1)


def test_golden_plans(port):
    """The restatement reproduces every golden reference plan (trees by hash)."""
    plans = golden("plans.json")
    specs = {"rectangles_2d_n2000": scene("rectangles_2d", 2000),
             "rectangles_3d_n1000": scene("rectangles_3d"), "maze_3d_n1500": scene("maze_3d", 1500),
             "rectangles_6d_n600": scene("rectangles_6d", 600), "cave_sim": scene("cave_sim"),
             "forest3d_n1000": P.forest_3d(3, 1000)}
    u = scene("rectangles_2d", 250)
    u.sampling_kind, u.seed = abi.SAMPLE_UNIFORM, 42
    specs["rectangles_2d_n250_uniform"] = u
    for name, spec in specs.items():
        rec = plans[name]
        o = oracle_instance(port, spec)
        assert o["coords"].shape[0] == rec["n"] and o["init"] == rec["init_index"]
        assert hexf(o["radius"]) == rec["radius"]
        assert sha(o["coords"]) == rec["coords_sha"] and o["goal_idx"].tolist() == rec["goal_idx"]
        assert sha(o["graph"].out_col) == rec["col_sha"]
        assert sha(o["graph"].out_cost) == rec["cost_sha"]
        for lam in (1.0, 0.5, 0.2):
            r = port.gmt_plan(spec, o["coords"], len(o["goal_idx"]), o["graph"], o["init"], lam,
                              o["radius"])
            p = rec["plans"][f"gmt_{lam}"]
            assert hexf(r.cost) == p["cost"] and r.iterations == p["iterations"], name
            assert r.total_collision_checks == p["checks"] and r.path_indices.tolist() == p["path"]
            assert r.group_sizes.tolist() == p["group_sizes"]
            assert r.nodes_added.tolist() == p["nodes_added"]
            assert r.collision_checks.tolist() == p["collision_checks"]
            assert sha(r.label) == p["label_sha"] and sha(r.tree_cost) == p["cost_sha"]
            assert sha(r.parent) == p["parent_sha"] and sha(r.iteration_added) == p["iter_added_sha"]
        f = port.fmt_plan(spec, o["coords"], len(o["goal_idx"]), o["graph"], o["init"])
        assert hexf(f.cost) == rec["plans"]["fmt"]["cost"]
        assert sha(f.tree_cost) == rec["plans"]["fmt"]["cost_sha"]


def test_sampling_semantics(port):
    """test_sampling.cpp:68-162 restated on the port."""
    e = P.ProblemSpec(dim=2, box_lo=np.zeros((0, 2)), box_hi=np.zeros((0, 2)),
                      goal_lo=np.zeros(2), goal_hi=np.ones(2), init=np.zeros(2), n=10)
    c, g = port.sample_free(e)
    for k in range(10):
        assert c[k, 0] == port.halton(k + 1, 2) and c[k, 1] == port.halton(k + 1, 3)
    assert g.tolist() == list(range(10))
    t = P.ProblemSpec(dim=2, box_lo=np.zeros((0, 2)), box_hi=np.zeros((0, 2)),
                      goal_lo=np.array([0.001, 0.001]), goal_hi=np.array([0.002, 0.002]),
                      init=np.zeros(2), n=50)
    c, g = port.sample_free(t)
    assert g.tolist() == [49] and abs(c[49, 0] - 0.0015) < 1e-15
    blocked = P.ProblemSpec(dim=2, box_lo=np.array([[0.55, 0.55]]), box_hi=np.array([[0.95, 0.95]]),
                            goal_lo=np.array([0.6, 0.6]), goal_hi=np.array([0.9, 0.9]),
                            init=np.zeros(2), n=50)
    with pytest.raises(GoalBlockedError):
        port.sample_free(blocked)
    full = P.ProblemSpec(dim=2, box_lo=np.array([[0.0, 0.0]]), box_hi=np.array([[1.0, 1.0]]),
                         goal_lo=np.array([0.6, 0.6]), goal_hi=np.array([0.9, 0.9]),
                         init=np.zeros(2), n=10)
    with pytest.raises(InfeasibleSamplingError):
        port.sample_free(full)


def test_segment_free_semantics(port):
    """Closed slab semantics (test_space.cpp:40-131)."""
    s = P.ProblemSpec(dim=2, box_lo=np.array([[0.4, 0.4]]), box_hi=np.array([[0.6, 0.6]]),
                      goal_lo=np.zeros(2), goal_hi=np.ones(2), init=np.zeros(2), n=1)
    assert not port.segment_free(s, [0.1, 0.5], [0.9, 0.5])    # crosses
    assert not port.segment_free(s, [0.1, 0.4], [0.9, 0.4])    # grazes a face: hit
    assert port.segment_free(s, [0.1, 0.39], [0.9, 0.39])
    assert not port.segment_free(s, [0.3, 0.3], [0.4, 0.4])    # touches a corner
    assert port.segment_free(s, [0.0, 0.0], [1.0, 0.0])        # cube boundary is free
    assert not port.segment_free(s, [0.5, 0.5], [0.5, 0.5])    # degenerate inside
    assert not port.segment_free(s, [0.1, 0.1], [1.1, 0.1])    # leaves the cube
    plane = P.ProblemSpec(dim=2, box_lo=np.array([[0.5, 0.0]]), box_hi=np.array([[0.5, 1.0]]),
                          goal_lo=np.zeros(2), goal_hi=np.ones(2), init=np.zeros(2), n=1)
    assert not port.segment_free(plane, [0.1, 0.3], [0.9, 0.7])  # zero-thickness plane blocks


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_port_equals_reference_random(port, ref, seed):
    """The reference's own random problems: port == reference bitwise."""
    rng = ref.rng(1000 + seed)
    for rep in range(8):
        dim = 2 + (rep + seed) % 3
        p = ref.random_problem(rng, dim=dim, with_obstacles=rep % 4 != 3, n_min=100, n_max=300)
        ptr, col, cost = ref.build_neighbor_graph(p["coords"], p["radius"], 4)
        pp, pc, pk = port.build_neighbor_graph(p["coords"], p["radius"])
        assert np.array_equal(ptr, pp) and np.array_equal(col, pc) and bits(cost) == bits(pk)
        g = Graph(p["coords"].shape[0], p["radius"], ptr, col, cost, dim=dim)
        # the port's sample_free reproduces the reference's uniform samples
        spec = p["spec"]
        for lam in (1.0, 0.4, 0.1):
            a = ref.gmt_plan(spec, p["coords"], len(p["goal_idx"]), g, p["init_index"], lam,
                             p["radius"], 3)
            b = port.gmt_plan(spec, p["coords"], len(p["goal_idx"]), g, p["init_index"], lam,
                              p["radius"])
            assert not abi.full_parity(a, b)
        a = ref.fmt_plan(spec, p["coords"], len(p["goal_idx"]), g, p["init_index"])
        b = port.fmt_plan(spec, p["coords"], len(p["goal_idx"]), g, p["init_index"])
        assert not abi.full_parity(a, b)


def test_python_random_problem_matches_reference(ref):
    """paper_1705_02403_b200.problem.random_problem_2d draws the same problems
    as the reference's make_random_problem (argument evaluation order
    included), so GPU tests can generate them without the reference."""
    rng_ref = ref.rng(4242)
    rng_py = P.Pcg32(4242)
    for _ in range(6):
        p = ref.random_problem(rng_ref, dim=2, n_min=80, n_max=200)
        s = P.random_problem_2d(rng_py, dim=2, n_min=80, n_max=200)
        assert np.array_equal(p["spec"].box_lo, s.box_lo) and np.array_equal(p["spec"].init, s.init)
        assert np.array_equal(p["spec"].goal_lo, s.goal_lo)
        c, _ = ref.sample_free(s)
        assert bits(c) == bits(p["coords"][: s.n])


@pytest.mark.parametrize("name", SCENE_NAMES)
def test_scene_instances_port_equals_reference(port, ref, name):
    spec = scene(name)
    a = oracle_instance(port, spec)
    b = oracle_instance(ref, spec)
    assert bits(a["coords"]) == bits(b["coords"]) and a["init"] == b["init"]
    assert a["graph"].same_as(b["graph"])
