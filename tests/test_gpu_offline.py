"""GPU parity of the offline phase: sample_free, append_init,
connection_radius, build_neighbor_graph and build_instance on the B200
against the compiled reference / the C restatement, bit for bit."""
import numpy as np
import pytest

from paper_1705_02403_b200 import abi, problem as P
from paper_1705_02403_b200.errors import (GoalBlockedError, InfeasibleSamplingError,
                                          InvalidInputError)
from helpers import SCENE_NAMES, bits, golden, oracle_instance, scene

pytestmark = pytest.mark.gpu


def _empty(dim, goal_lo, goal_hi, n=10, **kw):
    return P.ProblemSpec(dim=dim, box_lo=np.zeros((0, dim)), box_hi=np.zeros((0, dim)),
                         goal_lo=np.array(goal_lo, float), goal_hi=np.array(goal_hi, float),
                         init=np.full(dim, 0.05), n=n, **kw)


@pytest.mark.parametrize("name,n", [("rectangles_2d", 2000), ("maze_3d", 4000),
                                    ("rectangles_6d", 1000), ("cave_sim", None)])
def test_sample_free_halton_bitwise(ctx, port, name, n):
    spec = scene(name, n)
    want_c, want_g = port.sample_free(spec)
    got_c, got_g = ctx.sample_free(spec)
    assert bits(got_c) == bits(want_c)
    assert np.array_equal(got_g, want_g)


@pytest.mark.parametrize("seed", [1, 777, 4242, 2**63 + 5])
def test_sample_free_uniform_bitwise(ctx, ref, seed):
    spec = scene("rectangles_2d", 700)
    spec.sampling_kind = abi.SAMPLE_UNIFORM
    spec.seed = seed
    want_c, want_g = ref.sample_free(spec)
    got_c, got_g = ctx.sample_free(spec)
    assert bits(got_c) == bits(want_c)
    assert np.array_equal(got_g, want_g)


def test_sample_free_start_index(ctx, ref):
    spec = scene("maze_3d", 900)
    spec.start_index = 12345
    want_c, want_g = ref.sample_free(spec)
    got_c, got_g = ctx.sample_free(spec)
    assert bits(got_c) == bits(want_c) and np.array_equal(got_g, want_g)


def test_uniform_duplicates_in_one_dimension(ctx, ref):
    """d = 1 uniform draws collide often enough to exercise the exact
    duplicate rule (sampling.cpp:106)."""
    spec = _empty(1, [0.3], [0.31], n=3000)
    spec.sampling_kind = abi.SAMPLE_UNIFORM
    spec.seed = 99
    want_c, want_g = ref.sample_free(spec)
    got_c, got_g = ctx.sample_free(spec)
    assert bits(got_c) == bits(want_c) and np.array_equal(got_g, want_g)
    assert len(np.unique(got_c)) == len(got_c)


def test_goal_substitution_centre_and_fallback(ctx, ref):
    # tiny goal: centre substituted (test_sampling.cpp:128-137)
    spec = _empty(2, [0.001, 0.001], [0.002, 0.002], n=50)
    c, g = ctx.sample_free(spec)
    wc, wg = ref.sample_free(spec)
    assert bits(c) == bits(wc) and g.tolist() == wg.tolist() == [49]
    # centre blocked: rescaled Halton fallback (test_sampling.cpp:139-152)
    spec = _empty(2, [0.8, 0.8], [0.9, 0.9], n=20)
    spec.box_lo = np.array([[0.84, 0.84]])
    spec.box_hi = np.array([[0.86, 0.86]])
    c, g = ctx.sample_free(spec)
    wc, wg = ref.sample_free(spec)
    assert bits(c) == bits(wc) and g.tolist() == wg.tolist()


def test_sampling_errors(ctx):
    spec = _empty(2, [0.6, 0.6], [0.9, 0.9], n=50)
    spec.box_lo = np.array([[0.55, 0.55]])
    spec.box_hi = np.array([[0.95, 0.95]])
    with pytest.raises(GoalBlockedError):
        ctx.sample_free(spec)
    spec = _empty(2, [0.6, 0.6], [0.9, 0.9], n=10)
    spec.box_lo = np.array([[0.0, 0.0]])
    spec.box_hi = np.array([[1.0, 1.0]])
    with pytest.raises(InfeasibleSamplingError):
        ctx.sample_free(spec)
    spec = _empty(2, [0.6, 0.6], [0.9, 0.9], n=10)
    spec.start_index = 0
    with pytest.raises(InvalidInputError):
        ctx.sample_free(spec)


def test_append_init(ctx, ref):
    spec = _empty(2, [0.7, 0.7], [0.9, 0.9], n=25)
    c, g = ctx.sample_free(spec)
    c1, g1, i1 = ctx.append_init(c, g, [0.123, 0.456], spec.goal_lo, spec.goal_hi)
    assert i1 == 25 and c1.shape[0] == 26
    c2, g2, i2 = ctx.append_init(c1, g1, [0.123, 0.456], spec.goal_lo, spec.goal_hi)
    assert i2 == 25 and c2.shape[0] == 26
    c3, g3, i3 = ctx.append_init(c2, g2, [0.8, 0.8], spec.goal_lo, spec.goal_hi)
    assert i3 == 26 and g3[-1] == 26
    w3 = ref.append_init(c2, g2, [0.8, 0.8], spec.goal_lo, spec.goal_hi)
    assert bits(w3[0]) == bits(c3) and np.array_equal(w3[1], g3) and w3[2] == i3
    # exact duplicate of an existing sample is reused
    c4, g4, i4 = ctx.append_init(c3, g3, c3[7], spec.goal_lo, spec.goal_hi)
    assert i4 == 7 and c4.shape[0] == c3.shape[0]


def test_connection_radius_kats(ctx):
    from paper_1705_02403_b200.native import Context
    k = golden("kats.json")
    for d, n, eta, mu, hexv in k["radius"]:
        assert np.float64(Context.connection_radius(d, n, eta, mu)).tobytes().hex() == hexv
    for d, hexv in k["unit_ball"]:
        assert np.float64(Context.unit_ball_volume(d)).tobytes().hex() == hexv


@pytest.mark.parametrize("name,n,scale", [("rectangles_2d", 2000, 1.0), ("maze_3d", 4000, 1.0),
                                          ("rectangles_6d", 1500, 1.0), ("rectangles_6d", 1500, 0.4),
                                          ("cave_sim", None, 1.0), ("rectangles_3d", 3000, 2.0)])
def test_graph_bitwise(ctx, port, name, n, scale):
    spec = scene(name, n)
    coords, gidx = port.sample_free(spec)
    coords, gidx, _ = port.append_init(coords, gidx, spec.init, spec.goal_lo, spec.goal_hi)
    r = port.connection_radius(spec.dim, spec.n) * scale
    ptr, col, cost = port.build_neighbor_graph(coords, r)
    g = ctx.build_neighbor_graph(coords, r)
    assert np.array_equal(g.out_ptr, ptr)
    assert np.array_equal(g.out_col, col)
    assert bits(g.out_cost) == bits(cost)


def test_graph_12d_and_boundary_pairs(ctx, port):
    """12D extrusion (C4 stand-in shape) and pairs exactly at distance r:
    the inclusive `<= r` (graph.cpp:159) must hold bit for bit."""
    spec = P.extrude(scene("rectangles_2d", 600), 12)
    coords, _ = port.sample_free(spec)
    r = port.connection_radius(12, 600)
    ptr, col, cost = port.build_neighbor_graph(coords, r)
    g = ctx.build_neighbor_graph(coords, r)
    assert np.array_equal(g.out_col, col) and bits(g.out_cost) == bits(cost)
    pts = np.array([[0.0, 0.5], [0.1, 0.5], [0.25, 0.5], [0.35, 0.5], [0.5, 0.5]])
    for rr in (0.1, 0.15, 0.25, 0.2):
        ptr, col, cost = port.build_neighbor_graph(pts, rr)
        g = ctx.build_neighbor_graph(pts, rr)
        assert np.array_equal(g.out_ptr, ptr) and np.array_equal(g.out_col, col)


@pytest.mark.parametrize("name,n", [("rectangles_2d", 2000), ("maze_3d", 4000),
                                    ("rectangles_6d", 1000), ("cave_sim", None)])
def test_build_instance_matches_reference(ctx, ref, name, n):
    spec = scene(name, n)
    want = ref.instance_build(spec)
    wi = want.info()
    wc, wg, wptr, wcol, wcost = want.download(spec.dim)
    inst = ctx.build_instance(spec)
    assert (inst.n, inst.init_index, inst.num_edges, inst.goal_count) == (
        wi["n"], wi["init_index"], wi["num_edges"], wi["goal_count"])
    assert inst.radius == wi["radius"]
    c, g, graph = inst.download()
    assert bits(c) == bits(wc) and np.array_equal(g, wg)
    assert np.array_equal(graph.out_ptr, wptr) and np.array_equal(graph.out_col, wcol)
    assert bits(graph.out_cost) == bits(wcost)
    got = ctx.plan(inst, lam=spec.lam)
    assert not abi.full_parity(got, want.plan(spec.lam))


def test_golden_plans_end_to_end(ctx):
    """Reference known answers (tests/golden/plans.json, produced by the
    unmodified reference): device build_instance + gmt_plan reproduce the
    reference's trees (SHA-256 of label/cost/parent/iteration_added)."""
    import hashlib
    from helpers import scene as sc_
    plans = golden("plans.json")
    specs = {"rectangles_2d_n2000": sc_("rectangles_2d", 2000),
             "rectangles_3d_n1000": sc_("rectangles_3d"), "maze_3d_n1500": sc_("maze_3d", 1500),
             "rectangles_6d_n600": sc_("rectangles_6d", 600), "cave_sim": sc_("cave_sim"),
             "forest3d_n1000": P.forest_3d(3, 1000)}
    u = sc_("rectangles_2d", 250)
    u.sampling_kind, u.seed = abi.SAMPLE_UNIFORM, 42
    specs["rectangles_2d_n250_uniform"] = u
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    for name, spec in specs.items():
        rec = plans[name]
        inst = ctx.build_instance(spec)
        c, g, graph = inst.download()
        assert inst.n == rec["n"] and inst.num_edges == rec["num_edges"]
        assert sha(c) == rec["coords_sha"] and sha(graph.out_col) == rec["col_sha"]
        assert sha(graph.out_cost) == rec["cost_sha"] and g.tolist() == rec["goal_idx"]
        for lam in (1.0, 0.5, 0.2):
            r = ctx.plan(inst, lam=lam)
            p = rec["plans"][f"gmt_{lam}"]
            assert np.float64(r.cost).tobytes().hex() == p["cost"], name
            assert r.iterations == p["iterations"] and r.total_collision_checks == p["checks"]
            assert r.path_indices.tolist() == p["path"]
            assert r.group_sizes.tolist() == p["group_sizes"]
            assert sha(r.label) == p["label_sha"] and sha(r.tree_cost) == p["cost_sha"]
            assert sha(r.parent) == p["parent_sha"]
            assert sha(r.iteration_added) == p["iter_added_sha"]
        f = ctx.fmt_plan(inst)
        assert np.float64(f.cost).tobytes().hex() == rec["plans"]["fmt"]["cost"]
        assert sha(f.tree_cost) == rec["plans"]["fmt"]["cost_sha"]


@pytest.mark.parametrize("name,n", [("rectangles_2d", 2000), ("maze_3d", 1500)])
def test_build_instance_with_graph_cache(tmp_path, ctx, ref, name, n):
    """build_instance(p, workers, cache_file) (problem.cpp:336-363): the
    first device build misses, builds on the GPU and writes exactly the file
    the reference writes; the second hits and plans identically; a cache
    file written by the reference seeds a device instance."""
    from paper_1705_02403_b200 import native
    spec = scene(name, n)
    ours, theirs = str(tmp_path / "ours.gmtg"), str(tmp_path / "theirs.gmtg")
    a, hit_a = ctx.build_instance_cached(spec, ours)
    assert not hit_a
    ri = ref.instance_build_cached(spec, theirs)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    b, hit_b = ctx.build_instance_cached(spec, theirs)
    assert hit_b and b.num_edges == a.num_edges
    want = ri.plan(spec.lam)
    assert not abi.full_parity(ctx.plan(a, lam=spec.lam), want)
    assert not abi.full_parity(ctx.plan(b, lam=spec.lam), want)
    # an instance's graph saved explicitly is the same file again
    again = str(tmp_path / "again.gmtg")
    a.cache_save(again, native.problem_key(spec))
    assert open(again, "rb").read() == open(theirs, "rb").read()
