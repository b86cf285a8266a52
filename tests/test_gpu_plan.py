"""GPU parity of the online phase: gmt_plan / fmt_plan on the B200 against
the CPU oracle (the C restatement, itself pinned to the compiled reference)
on identical samples and graphs.  The bar is the reference's `same_tree`
(bitwise, tests/support/oracles.cpp:329-341) plus iterations, checks,
iteration_added and per-pass stats."""
import numpy as np
import pytest

from paper_1705_02403_b200 import abi, problem as P
from paper_1705_02403_b200.errors import InvalidInputError
from paper_1705_02403_b200.graph import Graph
from paper_1705_02403_b200.native import OPT_CLUSTER
from helpers import golden, oracle_instance, scene

pytestmark = pytest.mark.gpu

LAMBDAS = (1.0, 0.5, 0.2, 0.05)


def _assert_parity(a, b, what=""):
    bad = abi.full_parity(a, b)
    assert not bad, f"{what}: mismatch in {bad}: gpu={a} oracle={b}"


@pytest.mark.parametrize("name,n", [("rectangles_2d", 2000), ("rectangles_3d", 1500),
                                    ("maze_3d", 2000), ("rectangles_6d", 800),
                                    ("cave_sim", None)])
def test_scene_plans_match_oracle(ctx, port, name, n):
    spec = scene(name, n)
    o = oracle_instance(port, spec)
    inst = ctx.upload(spec, o["coords"], len(o["goal_idx"]), o["graph"])
    for lam in LAMBDAS:
        want = port.gmt_plan(spec, o["coords"], len(o["goal_idx"]), o["graph"], o["init"], lam,
                             o["radius"])
        got = ctx.plan(inst, o["init"], lam, o["radius"])
        _assert_parity(got, want, f"{name} lambda={lam}")


def test_c1_known_answer(ctx, port):
    """C1 = rectangles_2d n=2000: success, cost 1.690095...,
    21 iterations (22 passes), 1967 lazy checks, 1878 nodes reached."""
    spec = scene("rectangles_2d", 2000)
    o = oracle_instance(port, spec)
    inst = ctx.upload(spec, o["coords"], len(o["goal_idx"]), o["graph"])
    r = ctx.plan(inst, o["init"], 1.0, o["radius"])
    assert r.status == abi.PLAN_SUCCESS
    assert r.iterations == 21 and len(r.group_sizes) == 22
    assert r.total_collision_checks == 1967
    assert int((r.label != abi.LABEL_UNEXPLORED).sum()) == 1878
    rec = golden("plans.json")["rectangles_2d_n2000"]["plans"]["gmt_1.0"]
    assert np.float64(r.cost).tobytes().hex() == rec["cost"]
    assert r.path_indices.tolist() == rec["path"]


@pytest.mark.parametrize("cluster", [1, 2, 4, 8, 16])
def test_cluster_size_never_changes_result(ctx, port, cluster):
    """The worker-count invariance of test_planner.cpp:389-417, for the
    number of CTAs that cooperate on one query."""
    spec = scene("maze_3d", 1500)
    o = oracle_instance(port, spec)
    inst = ctx.upload(spec, o["coords"], len(o["goal_idx"]), o["graph"])
    want = port.gmt_plan(spec, o["coords"], len(o["goal_idx"]), o["graph"], o["init"], 0.7,
                         o["radius"])
    ctx.set_option(OPT_CLUSTER, cluster)
    try:
        got = ctx.plan(inst, o["init"], 0.7, o["radius"])
    finally:
        ctx.set_option(OPT_CLUSTER, 0)
    _assert_parity(got, want, f"cluster={cluster}")


def test_random_reference_problems(ctx, ref):
    """The reference's own seeded problems (make_random_problem,
    oracles.cpp:258-327): uniform samples, 2-6 boxes, 2-4 dims, several
    lambdas, GPU == unmodified reference bit for bit."""
    rng = ref.rng(20240601)
    compared = 0
    for rep in range(24):
        dim = 2 + rep % 3
        p = ref.random_problem(rng, dim=dim, with_obstacles=rep % 5 != 4, n_min=120, n_max=400)
        ptr, col, cost = ref.build_neighbor_graph(p["coords"], p["radius"])
        g = Graph(p["coords"].shape[0], p["radius"], ptr, col, cost, dim=dim)
        inst = ctx.upload(p["spec"], p["coords"], len(p["goal_idx"]), g)
        for lam in (1.0, 0.35):
            want = ref.gmt_plan(p["spec"], p["coords"], len(p["goal_idx"]), g, p["init_index"], lam,
                                p["radius"])
            got = ctx.plan(inst, p["init_index"], lam, p["radius"])
            _assert_parity(got, want, f"rep={rep} lambda={lam}")
            compared += 1
    assert compared == 48


def test_plan_host_drop_in(ctx, ref):
    """gmt_plan with every input in host memory (the C++ shim's call)."""
    spec = scene("rectangles_3d", 1200)
    o = oracle_instance(ref, spec)
    for lam in (1.0, 0.3):
        want = ref.gmt_plan(spec, o["coords"], len(o["goal_idx"]), o["graph"], o["init"], lam,
                            o["radius"])
        got = ctx.plan_host(spec, o["coords"], len(o["goal_idx"]), o["graph"], o["init"], lam,
                            o["radius"])
        _assert_parity(got, want, f"plan_host lambda={lam}")


def test_fmt_plan_matches_reference(ctx, ref):
    spec = scene("rectangles_2d", 600)
    o = oracle_instance(ref, spec)
    inst = ctx.upload(spec, o["coords"], len(o["goal_idx"]), o["graph"])
    want = ref.fmt_plan(spec, o["coords"], len(o["goal_idx"]), o["graph"], o["init"])
    got = ctx.fmt_plan(inst, o["init"])
    _assert_parity(got, want, "fmt")


def test_tiny_lambda_reproduces_fmt(ctx, ref):
    """test_planner.cpp:174-211: with delta below half the smallest cost gap
    every group is a singleton and the GMT* tree equals FMT*'s bit for bit."""
    rng = ref.rng(8080)
    compared = 0
    for _ in range(8):
        p = ref.random_problem(rng, n_min=120, n_max=250)
        ptr, col, cost = ref.build_neighbor_graph(p["coords"], p["radius"])
        g = Graph(p["coords"].shape[0], p["radius"], ptr, col, cost, dim=2)
        inst = ctx.upload(p["spec"], p["coords"], len(p["goal_idx"]), g)
        fmt = ctx.fmt_plan(inst, p["init_index"])
        if fmt.status != abi.PLAN_SUCCESS:
            continue
        c = np.sort(fmt.tree_cost[np.isfinite(fmt.tree_cost)])
        gaps = np.diff(c)
        gaps = gaps[gaps > 0]
        if len(gaps) == 0:
            continue
        lam = min(1.0, 0.49 * gaps.min() / p["radius"])
        gmt = ctx.plan(inst, p["init_index"], lam, p["radius"])
        assert all(s <= 1 for s in gmt.group_sizes)
        assert abi.same_tree(gmt, fmt)
        compared += 1
    assert compared >= 3


def test_edge_cases(ctx, ref):
    # init already inside the goal (test_planner.cpp:89-111)
    spec = P.ProblemSpec(dim=2, box_lo=np.zeros((0, 2)), box_hi=np.zeros((0, 2)),
                         goal_lo=np.array([0.4, 0.4]), goal_hi=np.array([0.6, 0.6]),
                         init=np.array([0.5, 0.5]), n=1)
    coords, gidx = ref.sample_free(spec)
    coords, gidx, ii = ref.append_init(coords, gidx, spec.init, spec.goal_lo, spec.goal_hi)
    ptr, col, cost = ref.build_neighbor_graph(coords, 0.3)
    g = Graph(coords.shape[0], 0.3, ptr, col, cost, dim=2)
    inst = ctx.upload(spec, coords, len(gidx), g)
    r = ctx.plan(inst, ii, 1.0, 0.3)
    assert r.status == abi.PLAN_SUCCESS and r.cost == 0.0 and r.iterations == 0
    assert r.path_indices.tolist() == [ii] and r.total_collision_checks == 0

    # colliding init -> infeasible input with an EMPTY tree (planner.cpp:108)
    spec2 = P.ProblemSpec(dim=2, box_lo=np.array([[0.4, 0.4]]), box_hi=np.array([[0.6, 0.6]]),
                          goal_lo=np.array([0.8, 0.8]), goal_hi=np.array([0.9, 0.9]),
                          init=np.array([0.5, 0.5]), n=50)
    coords, gidx = ref.sample_free(spec2)
    coords, gidx, ii = ref.append_init(coords, gidx, spec2.init, spec2.goal_lo, spec2.goal_hi)
    ptr, col, cost = ref.build_neighbor_graph(coords, 0.3)
    g = Graph(coords.shape[0], 0.3, ptr, col, cost, dim=2)
    inst = ctx.upload(spec2, coords, len(gidx), g)
    r = ctx.plan(inst, ii, 1.0, 0.3)
    assert r.status == abi.PLAN_INFEASIBLE_INPUT and len(r.label) == 0 and r.cost == np.inf
    # no goal samples -> infeasible input
    inst0 = ctx.upload(spec2, coords, 0, g)
    assert ctx.plan(inst0, 0, 1.0, 0.3).status == abi.PLAN_INFEASIBLE_INPUT

    # validation throws InvalidInputError (test_planner.cpp:153-172)
    for lam, rad, init in ((0.0, 0.3, ii), (1.5, 0.3, ii), (1.0, 0.25, ii), (1.0, 0.3, -1),
                           (1.0, 0.3, coords.shape[0])):
        with pytest.raises(InvalidInputError):
            ctx.plan(inst, init, lam, rad)


def test_sealed_goal_pocket_exhausts_open_set(ctx, ref):
    spec = P.ProblemSpec(dim=2, box_lo=np.array([[0.6, 0.6], [0.6, 0.6]]),
                         box_hi=np.array([[1.0, 0.7], [0.7, 1.0]]),
                         goal_lo=np.array([0.8, 0.8]), goal_hi=np.array([0.9, 0.9]),
                         init=np.array([0.1, 0.1]), n=800)
    o = oracle_instance(ref, spec)
    inst = ctx.upload(spec, o["coords"], len(o["goal_idx"]), o["graph"])
    got = ctx.plan(inst, o["init"], 1.0, o["radius"])
    want = ref.gmt_plan(spec, o["coords"], len(o["goal_idx"]), o["graph"], o["init"], 1.0,
                        o["radius"])
    assert got.status == abi.PLAN_FAILURE_OPEN_EMPTY and got.iterations > 0
    _assert_parity(got, want, "sealed")


def test_batch_equals_single(ctx, port):
    specs = [P.random_forest_query(7, q, n=600) for q in range(6)]
    insts, wants = [], []
    for s in specs:
        o = oracle_instance(port, s)
        insts.append(ctx.upload(s, o["coords"], len(o["goal_idx"]), o["graph"]))
        wants.append(port.gmt_plan(s, o["coords"], len(o["goal_idx"]), o["graph"], o["init"], 1.0,
                                   o["radius"]))
        insts[-1].init_index_ = o["init"]
    b = ctx.batch(insts, 1.0, init_index=[i.init_index_ for i in insts])
    b.launch()
    sums = b.summaries()
    for q in range(len(specs)):
        got = b.result(q)
        _assert_parity(got, wants[q], f"batch q={q}")
        assert sums[q].status == wants[q].status and sums[q].iterations == wants[q].iterations


def test_plan_batch_host_pipelined_matches_reference(ctx, port):
    """The batched drop-in with host buffers (gmt_plan_batch_host): 130
    queries go through the chunked copy/solve pipeline; every summary, path
    and tree equals the oracle's plan of the same query."""
    from paper_1705_02403_b200.native import PackedBatch, plan_batch_host
    entries, wants = [], []
    for q in range(130):
        s = P.random_forest_query(77, q, n=300)
        o = oracle_instance(port, s)
        entries.append((s, o["coords"], len(o["goal_idx"]), o["graph"], o["init"]))
        wants.append(port.gmt_plan(s, o["coords"], len(o["goal_idx"]), o["graph"], o["init"], 1.0,
                                   o["radius"]))
    pb = PackedBatch(entries, want_tree=True)
    plan_batch_host(ctx, pb, 1.0)
    for q, w in enumerate(wants):
        got = pb.query_result(q)
        assert abi.same_tree(got, w), q
        assert got.iterations == w.iterations and got.total_collision_checks == w.total_collision_checks
        assert np.array_equal(got.iteration_added, w.iteration_added)
