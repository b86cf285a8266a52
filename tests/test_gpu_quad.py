"""GPU parity of the 12D linearised-quadrotor path: device steering costs,
durations, graphs and waypoints equal the oracle's statement of the model
bit for bit, and device plans on device-built quadrotor instances
(trajectories regenerated in the solve kernel) equal the unmodified
reference's gmt_plan on the same graph injected with cached polylines."""
import numpy as np
import pytest

from paper_1705_02403_b200 import abi, problem as P
from paper_1705_02403_b200.native import OPT_CLUSTER
from helpers import bits
from test_quad import _pairs, _params, small_scene

pytestmark = pytest.mark.gpu


def test_device_quad_costs_bitwise(ctx, port):
    p = _params()
    pairs = _pairs(3, 1500) + _pairs(4, 300, spread=1.0)
    pairs.append((np.full(12, 0.5), np.full(12, 0.5)))
    y = np.full(12, 0.5)
    y[3] = 0.9
    pairs.append((y, y))
    x0 = np.array([q[0] for q in pairs])
    x1 = np.array([q[1] for q in pairs])
    c, t = ctx.quad_costs(x0, x1, p)
    want = np.array([port.quad_cost(a, b, p) for a, b in pairs])
    assert bits(c) == bits(np.ascontiguousarray(want[:, 0]))
    assert bits(t) == bits(np.ascontiguousarray(want[:, 1]))


@pytest.mark.parametrize("n,r", [(300, 5.0), (500, 4.5)])
def test_device_quad_graph_bitwise(ctx, port, n, r):
    spec = P.quad_scene(5, n, radius=r)
    qp = spec.quad_params()
    c, g = port.sample_free(spec)
    c, g, ii = port.append_init(c, g, spec.init, spec.goal_lo, spec.goal_hi)
    G = ctx.build_quad_graph(c, qp, r, paths=True)
    W = port.quad_graph(c, r, qp)
    assert len(W.out_col) > 0
    assert np.array_equal(G.out_ptr, W.out_ptr) and np.array_equal(G.out_col, W.out_col)
    assert bits(G.out_cost) == bits(W.out_cost) and bits(G.out_tau) == bits(W.out_tau)
    assert np.array_equal(G.in_ptr, W.in_ptr) and np.array_equal(G.in_col, W.in_col)
    assert bits(G.in_cost) == bits(W.in_cost) and np.array_equal(G.in_path, W.in_path)
    assert bits(G.path_pts) == bits(W.path_pts)


@pytest.mark.parametrize("seed,n,r,lam", [(5, 400, 4.5, 1.0), (5, 400, 4.5, 0.3), (6, 300, 5.0, 0.5),
                                          (7, 600, 4.2, 1.0)])
def test_device_quad_instance_plans_match_reference(ctx, port, ref, seed, n, r, lam):
    spec = small_scene(seed, n, r)
    inst = ctx.build_instance(spec)          # samples + quadrotor graph on the device
    c, g, _ = inst.download()
    wc, wg = port.sample_free(spec)
    wc, wg, ii = port.append_init(wc, wg, spec.init, spec.goal_lo, spec.goal_hi)
    assert bits(c) == bits(wc) and inst.init_index == ii
    G = port.quad_graph(wc, r, spec.quad_params())   # cached polylines for the reference
    want = ref.gmt_plan(spec, wc, len(wg), G, ii, lam, r)
    got = ctx.plan(inst, lam=lam)            # kernel regenerates the polylines
    assert not abi.full_parity(got, want), abi.full_parity(got, want)
    up = ctx.upload(spec, wc, len(wg), G)
    assert not abi.full_parity(ctx.plan(up, ii, lam, r), want)


def test_quad_full_size_plan_matches_explicit_path_route(ctx):
    """C4 at full size (n = 8000): the device-built instance (implicit
    trajectories) and the same graph downloaded and re-uploaded with its
    waypoint polylines (explicit paths, the reference's route) plan
    identically, for several cluster sizes."""
    spec = P.quad_scene()
    inst = ctx.build_instance(spec)
    base = ctx.plan(inst)
    assert base.status == abi.PLAN_SUCCESS
    c, g, _ = inst.download()
    G = ctx.build_quad_graph(c, spec.quad_params(), spec.radius_override, paths=True)
    up = ctx.upload(spec, c, len(g), G)
    assert not abi.full_parity(ctx.plan(up, inst.init_index, spec.lam, spec.radius_override), base)
    for cluster in (1, 4, 16):
        ctx.set_option(OPT_CLUSTER, cluster)
        try:
            assert not abi.full_parity(ctx.plan(inst), base)
        finally:
            ctx.set_option(OPT_CLUSTER, 0)


def test_quad_batch_queries(ctx):
    specs = [small_scene(s, 600, 4.5) for s in (5, 8, 22)]
    insts = [ctx.build_instance(s) for s in specs]
    b = ctx.batch(insts, 1.0)
    b.launch()
    for q, inst in enumerate(insts):
        assert not abi.full_parity(b.result(q), ctx.plan(inst))


@pytest.mark.parametrize("model", ["quad", "di"])
def test_waypoint_tables_equal_regeneration(ctx, monkeypatch, model):
    """The build-time per-in-edge waypoint tables (sample.cu, solve.cu
    kino_table_kernel) against regenerating each checked trajectory in the
    solve (GMT_KINO_TABLES=0): full plans bit for bit, single CTA and
    cluster shapes, lambda 1 and 0.5."""
    spec = P.quad_scene(5, 2500) if model == "quad" else P.di_forest(3, 1500)
    got = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("GMT_KINO_TABLES", mode)
        inst = ctx.build_instance(spec)
        for cs in (1, 8):
            ctx.set_option(OPT_CLUSTER, cs)
            for lam in (1.0, 0.5):
                got[mode, cs, lam] = ctx.plan(inst, lam=lam)
        ctx.set_option(OPT_CLUSTER, 0)
    for (mode, cs, lam), r in got.items():
        if mode == "1":
            assert not abi.full_parity(r, got["0", cs, lam]), (cs, lam)
    assert got["1", 1, 1.0].total_collision_checks > 0
