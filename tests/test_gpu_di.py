"""GPU parity of the 6D double-integrator path: device steering costs,
durations, graphs and waypoints equal the oracle's statement of the model
bit for bit, and device plans on device-built DI instances (trajectories
regenerated in the solve kernel) equal the unmodified reference's gmt_plan
on the same graph injected with cached polylines."""
import numpy as np
import pytest

from paper_1705_02403_b200 import abi, problem as P
from paper_1705_02403_b200.native import OPT_CLUSTER
from helpers import bits
from test_di import _pairs

pytestmark = pytest.mark.gpu


def _params(spec=None):
    p = abi.DiParams()
    p.vmax, p.weight, p.segments, p.reserved = 0.5, 1.0, 8, 0
    return p if spec is None else spec.di_params()


def test_device_di_costs_bitwise(ctx, port):
    pairs = _pairs(3, 2000)
    pairs.append((np.full(6, 0.5), np.full(6, 0.5)))
    pairs.append((np.array([0.1, 0.2, 0.3, 0.9, 0.1, 0.5]),) * 2)
    x0 = np.array([p[0] for p in pairs])
    x1 = np.array([p[1] for p in pairs])
    c, t = ctx.di_costs(x0, x1, _params())
    want = np.array([port.di_cost(a, b) for a, b in pairs])
    assert bits(c) == bits(np.ascontiguousarray(want[:, 0]))
    assert bits(t) == bits(np.ascontiguousarray(want[:, 1]))


@pytest.mark.parametrize("n,r", [(600, 2.4), (1200, 2.0)])
def test_device_di_graph_bitwise(ctx, port, n, r):
    spec = P.di_forest(3, n, radius=r)
    c, g = port.sample_free(spec)
    c, g, ii = port.append_init(c, g, spec.init, spec.goal_lo, spec.goal_hi)
    G = ctx.build_di_graph(c, _params(), r, paths=True)
    W = port.di_graph(c, r)
    assert np.array_equal(G.out_ptr, W.out_ptr) and np.array_equal(G.out_col, W.out_col)
    assert bits(G.out_cost) == bits(W.out_cost) and bits(G.out_tau) == bits(W.out_tau)
    assert np.array_equal(G.in_ptr, W.in_ptr) and np.array_equal(G.in_col, W.in_col)
    assert bits(G.in_cost) == bits(W.in_cost) and np.array_equal(G.in_path, W.in_path)
    assert bits(G.path_pts) == bits(W.path_pts)


@pytest.mark.parametrize("n,r,lam", [(600, 2.4, 1.0), (900, 2.2, 0.5), (900, 2.2, 0.2)])
def test_device_di_instance_plans_match_reference(ctx, port, ref, n, r, lam):
    spec = P.di_forest(3, n, radius=r)
    inst = ctx.build_instance(spec)          # samples + DI graph on the device
    c, g, _ = inst.download()
    wc, wg = port.sample_free(spec)
    wc, wg, ii = port.append_init(wc, wg, spec.init, spec.goal_lo, spec.goal_hi)
    assert bits(c) == bits(wc) and inst.init_index == ii
    G = port.di_graph(wc, r)                 # cached polylines for the reference
    want = ref.gmt_plan(spec, wc, len(wg), G, ii, lam, r)
    got = ctx.plan(inst, lam=lam)            # kernel regenerates the polylines
    assert not abi.full_parity(got, want), abi.full_parity(got, want)
    # the explicit-path route (uploaded graph) agrees too
    up = ctx.upload(spec, wc, len(wg), G)
    assert not abi.full_parity(ctx.plan(up, ii, lam, r), want)


@pytest.mark.parametrize("cluster", [1, 4, 16])
def test_di_cluster_invariance(ctx, port, cluster):
    spec = P.di_forest(5, 800, radius=2.3)
    inst = ctx.build_instance(spec)
    base = ctx.plan(inst)
    ctx.set_option(OPT_CLUSTER, cluster)
    try:
        got = ctx.plan(inst)
    finally:
        ctx.set_option(OPT_CLUSTER, 0)
    assert not abi.full_parity(got, base)


def test_di_batch_queries(ctx, port):
    specs = [P.random_di_query(11, q, n=500, radius=2.5) for q in range(4)]
    insts = [ctx.build_instance(s) for s in specs]
    b = ctx.batch(insts, 1.0)
    b.launch()
    for q, (s, inst) in enumerate(zip(specs, insts)):
        assert not abi.full_parity(b.result(q), ctx.plan(inst))


@pytest.mark.parametrize("lam", [1.0, 0.5])
def test_di_boxes_with_velocity_extent(ctx, port, ref, lam):
    """Boxes that do not span the whole velocity range (the lazy check then
    tests the trajectory's velocity coordinates against them too): device
    plans equal the reference on the injected graph."""
    spec = P.di_forest(7, 700, radius=2.3)
    lo, hi = spec.box_lo.copy(), spec.box_hi.copy()
    lo[::2, 3] = 0.55        # every other pillar only blocks fast +x motion
    hi[1::3, 4] = 0.45       # some only block -y motion
    spec.box_lo, spec.box_hi = lo, hi
    # a few velocity-space slabs over the whole workspace
    spec.box_lo = np.vstack([spec.box_lo, [[0, 0, 0, 0.93, 0, 0], [0, 0, 0, 0, 0, 0.0]]])
    spec.box_hi = np.vstack([spec.box_hi, [[1, 1, 1, 1.0, 1, 1], [1, 1, 1, 1, 1, 0.04]]])
    inst = ctx.build_instance(spec)
    c, g, _ = inst.download()
    wc, wg = port.sample_free(spec)
    wc, wg, ii = port.append_init(wc, wg, spec.init, spec.goal_lo, spec.goal_hi)
    assert bits(c) == bits(wc)
    G = port.di_graph(wc, 2.3)
    want = ref.gmt_plan(spec, wc, len(wg), G, ii, lam, 2.3)
    got = ctx.plan(inst, lam=lam)
    assert not abi.full_parity(got, want), abi.full_parity(got, want)
    b = ctx.batch([inst], lam)
    b.launch()
    assert not abi.full_parity(b.result(0), want)
