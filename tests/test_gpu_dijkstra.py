"""GPU parity of dijkstra_oracle (planner.cpp:264-334; SURVEY.md §8(f) row
4): the device's eager edge checks + exact Dijkstra equal the unmodified
reference bit for bit -- tree (labels, costs, parents), path, cost, pops
(iterations) and the eager check count -- on uploaded and device-built
instances, Euclidean (symmetric checks) and directed (cached-path and
kinodynamic) graphs, and the infeasible case."""
import numpy as np
import pytest

from paper_1705_02403_b200 import abi, problem as P
from helpers import oracle_instance, scene
from test_quad import small_scene

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,n", [("rectangles_2d", 600), ("rectangles_2d", 2000), ("maze_3d", 1500),
                                    ("rectangles_6d", 500), ("cave_sim", None)])
def test_device_dijkstra_matches_reference(ctx, port, ref, name, n):
    spec = scene(name, n)
    o = oracle_instance(port, spec)
    want = ref.dijkstra_oracle(spec, o["coords"], len(o["goal_idx"]), o["graph"], o["init"])
    up = ctx.upload(spec, o["coords"], len(o["goal_idx"]), o["graph"])
    got = ctx.dijkstra_oracle(up, o["init"])
    assert not abi.full_parity(got, want), abi.full_parity(got, want)
    built = ctx.build_instance(spec)
    assert not abi.full_parity(ctx.dijkstra_oracle(built), want)
    # the oracle's cost lower-bounds GMT*'s (it checks every edge eagerly)
    g = ctx.plan(built, lam=1.0)
    if want.status == abi.PLAN_SUCCESS and g.status == abi.PLAN_SUCCESS:
        assert want.cost <= g.cost + 1e-12


def test_device_dijkstra_forest_and_infeasible(ctx, port, ref):
    spec = P.forest_3d(3, 1200)
    o = oracle_instance(port, spec)
    want = ref.dijkstra_oracle(spec, o["coords"], len(o["goal_idx"]), o["graph"], o["init"])
    up = ctx.upload(spec, o["coords"], len(o["goal_idx"]), o["graph"])
    assert not abi.full_parity(ctx.dijkstra_oracle(up, o["init"]), want)
    # init inside an obstacle: empty tree, infeasible_input
    blocked = spec.with_n(200)
    blocked.box_lo = np.vstack([blocked.box_lo, blocked.init - 0.01])
    blocked.box_hi = np.vstack([blocked.box_hi, blocked.init + 0.01])
    ob = oracle_instance(port, blocked)
    want = ref.dijkstra_oracle(blocked, ob["coords"], len(ob["goal_idx"]), ob["graph"], ob["init"])
    up = ctx.upload(blocked, ob["coords"], len(ob["goal_idx"]), ob["graph"])
    got = ctx.dijkstra_oracle(up, ob["init"])
    assert got.status == want.status == abi.PLAN_INFEASIBLE_INPUT
    assert not abi.full_parity(got, want)


@pytest.mark.parametrize("n,r", [(600, 2.4), (900, 2.2)])
def test_device_dijkstra_double_integrator(ctx, port, ref, n, r):
    """Directed graph: every edge is its own motion; the device-built
    instance regenerates each out-edge trajectory, the reference checks the
    cached polylines of the same graph."""
    spec = P.di_forest(3, n, radius=r)
    inst = ctx.build_instance(spec)
    wc, wg = port.sample_free(spec)
    wc, wg, ii = port.append_init(wc, wg, spec.init, spec.goal_lo, spec.goal_hi)
    G = port.di_graph(wc, r)
    want = ref.dijkstra_oracle(spec, wc, len(wg), G, ii)
    assert not abi.full_parity(ctx.dijkstra_oracle(inst), want)
    up = ctx.upload(spec, wc, len(wg), G)
    assert not abi.full_parity(ctx.dijkstra_oracle(up, ii), want)


def test_device_dijkstra_quadrotor(ctx, port, ref):
    spec = small_scene(5, 400, 4.5)
    inst = ctx.build_instance(spec)
    wc, wg = port.sample_free(spec)
    wc, wg, ii = port.append_init(wc, wg, spec.init, spec.goal_lo, spec.goal_hi)
    G = port.quad_graph(wc, 4.5, spec.quad_params())
    want = ref.dijkstra_oracle(spec, wc, len(wg), G, ii)
    assert not abi.full_parity(ctx.dijkstra_oracle(inst), want)
