"""Dubins-airplane steering on the device (
dubins.cpp:84-167, steering.cpp:53-121).  The reference computes the word
parameters with glibc's sin/cos/atan2/acos, which are not correctly rounded
(0.06-0.15 % of results differ from the correctly rounded value, measured
here), so device costs are checked to a few ulps rather than bit for bit;
the graph's edge set, the samples and every planner result over the
reference's own Dubins graph (cached paths, uploaded) are checked exactly."""
import numpy as np
import pytest

from paper_1705_02403_b200 import abi, native, problem as P
from helpers import forest_dubins

pytestmark = pytest.mark.gpu


def _params(rho=0.08, step=0.0, planar=False):
    p = abi.DubinsParams()
    p.rho, p.discretization_step, p.planar_cost_only, p.reserved = rho, step, int(planar), 0
    return p


@pytest.mark.parametrize("dim,planar", [(2, False), (3, False), (3, True)])
def test_dubins_costs_within_ulps(ctx, ref, dim, planar):
    rng = np.random.default_rng(dim * 10 + planar)
    m = 4000
    x0 = rng.random((m, dim + 1))
    x1 = rng.random((m, dim + 1))
    x0[:, dim] *= 2 * np.pi
    x1[:, dim] *= 2 * np.pi
    x1[:5] = x0[:5]  # degenerate pairs
    p = _params(0.08, 0.0, planar)
    c, s = ctx.dubins_costs(x0, x1, dim, p)
    rc, rs = ref.dubins_costs(x0, x1, dim, p)
    assert np.all(c[:5] == 0) and np.all(s[:5] == 0) and np.all(rs[:5] == 0)
    rel = np.abs(c - rc) / np.maximum(rc, 1e-300)
    assert rel.max() < 1e-12, rel.max()
    assert np.mean(c == rc) > 0.5          # most costs are bit-identical
    assert np.mean(s == rs) > 0.999         # ceil(Lp / step) flips only at boundaries


def test_forest_dubins_graph_and_plan(ctx, ref):
    spec = forest_dubins()
    ri = ref.instance_build(spec)
    coords, gidx, G = ri.graph(2)
    inst = ctx.build_instance(spec)
    info = ri.info()
    assert (inst.n, inst.init_index, inst.goal_count) == (info["n"], info["init_index"], info["goal_count"])
    c, g, dev = inst.download()
    assert c.tobytes() == coords.tobytes()          # samples (with headings) bit for bit
    # the edge set is the reference's up to pairs whose cost lies within
    # rounding of r (glibc's transcendentals vs the device's):
    # every mismatched pair's reference cost must be within 1e-12 of r
    pairs = []
    for u in range(inst.n):
        a = set(dev.out_col[dev.out_ptr[u]:dev.out_ptr[u + 1]].tolist())
        b = set(G.out_col[G.out_ptr[u]:G.out_ptr[u + 1]].tolist())
        pairs += [(u, v) for v in sorted(a ^ b)]
    mism = len(pairs)
    if pairs:
        x0 = np.array([coords[u] for u, _ in pairs])
        x1 = np.array([coords[v] for _, v in pairs])
        rc, _ = ref.dubins_costs(x0, x1, 2, spec.dubins_params())
        r = info["radius"]
        assert np.all(np.abs(rc - r) <= 1e-12 * r), (pairs, rc, r)
    if mism == 0:
        rel = np.abs(dev.out_cost - G.out_cost) / np.maximum(G.out_cost, 1e-300)
        assert rel.max() < 1e-12
    # planning on the device-built graph: same outcome, cost to rounding
    want = ri.plan(spec.lam)
    got = ctx.plan(inst, lam=spec.lam)
    assert got.status == want.status == abi.PLAN_SUCCESS
    assert abs(got.cost - want.cost) <= 1e-9 * want.cost
    # exact pin: the reference's own Dubins graph (cached paths) uploaded
    up = ctx.upload(spec, coords, len(gidx), G)
    ii = info["init_index"]
    assert not abi.full_parity(ctx.plan(up, ii, spec.lam, info["radius"]), want)
    assert not abi.full_parity(ctx.fmt_plan(up, ii), ref.fmt_plan(spec, coords, len(gidx), G, ii))
    assert not abi.full_parity(ctx.dijkstra_oracle(up, ii),
                               ref.dijkstra_oracle(spec, coords, len(gidx), G, ii))


def test_dubins_graph_cache_with_reference(tmp_path, ctx, ref):
    """GMTG v1 files for Dubins problems (graph.cpp:245-343): the header and
    key match the reference's; the reference loads our file; a reference
    file seeds a device instance with the reference's exact costs (paths
    recomputed on load, as the reference does), which then plans exactly
    like the reference; an instance saved again is the same file."""
    spec = forest_dubins()
    key = native.problem_key(spec)
    assert key == ref.problem_key(spec)
    ours, theirs, again = (str(tmp_path / f) for f in ("ours.gmtg", "theirs.gmtg", "again.gmtg"))
    a, hit_a = ctx.build_instance_cached(spec, ours)
    assert not hit_a
    ri = ref.instance_build_cached(spec, theirs)
    ob, tb = open(ours, "rb").read(), open(theirs, "rb").read()
    header = 4 + 4 + 8 + 4 + 8 + 1 + 8 + 8 + 1
    assert ob[:header] == tb[:header] and len(ob) == len(tb)  # same edge set; costs to a few ulps
    coords, gidx, G = ri.graph(2)
    _, _, ga = a.download()
    assert np.array_equal(ga.out_col, G.out_col)
    # the reference's build_instance loads our file: its graph carries our costs
    _, _, G2 = ref.instance_build_cached(spec, ours).graph(2)
    assert G2.out_cost.tobytes() == ga.out_cost.tobytes()
    b, hit_b = ctx.build_instance_cached(spec, theirs)
    assert hit_b and b.num_edges == a.num_edges
    _, _, gb = b.download()
    assert gb.out_cost.tobytes() == G.out_cost.tobytes()  # the reference's costs, exactly
    assert not abi.full_parity(ctx.plan(b, lam=spec.lam), ri.plan(spec.lam))
    b.cache_save(again, key)
    assert open(again, "rb").read() == tb
    # a Dubins file is a miss for the Euclidean problem over the same scene, and vice versa
    eu = forest_dubins()
    eu.steering = abi.STEER_EUCLIDEAN
    _, hit_e = ctx.build_instance_cached(eu, theirs)
    assert not hit_e
