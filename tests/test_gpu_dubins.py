"""Dubins-airplane steering on the device (
dubins.cpp:84-167, steering.cpp:53-121), bit for bit against the reference:
the word parameters and path poses go through glibc's sin / cos / atan2 /
acos and the prune through its hypot, which the device evaluates with the
restatements of glibc's own routines (csrc/libm_port.cuh, pinned on the
host by tests/test_libm_port.py).  Costs, segment counts, the graph's edge
set and costs, the samples, every planner result on the device-built graph
and on the reference's own graph (uploaded), and the GMTG cache files."""
import numpy as np
import pytest

from paper_1705_02403_b200 import abi, native, problem as P
from helpers import forest_dubins

pytestmark = pytest.mark.gpu


def _params(rho=0.08, step=0.0, planar=False):
    p = abi.DubinsParams()
    p.rho, p.discretization_step, p.planar_cost_only, p.reserved = rho, step, int(planar), 0
    return p


@pytest.mark.parametrize("dim,planar,rho", [(2, False, 0.08), (3, False, 0.08), (3, True, 0.08),
                                            (2, False, 0.3), (3, False, 0.01)])
def test_dubins_costs_bitwise(ctx, ref, dim, planar, rho):
    rng = np.random.default_rng(dim * 10 + planar + int(rho * 100))
    m = 20000
    x0 = rng.random((m, dim + 1))
    x1 = rng.random((m, dim + 1))
    x0[:, dim] *= 2 * np.pi
    x1[:, dim] *= 2 * np.pi
    x1[:5] = x0[:5]  # degenerate pairs
    x1[5:400, :dim] = x0[5:400, :dim] + rng.normal(0, 1e-3, (395, dim))  # short hops (RLR / LRL words)
    x1[400:600, dim] = x0[400:600, dim]                                     # equal headings
    p = _params(rho, 0.0, planar)
    c, s = ctx.dubins_costs(x0, x1, dim, p)
    rc, rs = ref.dubins_costs(x0, x1, dim, p)
    assert np.all(c[:5] == 0) and np.all(s[:5] == 0)
    assert c.tobytes() == rc.tobytes(), int(np.sum(c != rc))
    assert np.array_equal(s, rs)


def test_forest_dubins_graph_and_plan(ctx, ref):
    spec = forest_dubins()
    ri = ref.instance_build(spec)
    coords, gidx, G = ri.graph(2)
    inst = ctx.build_instance(spec)
    info = ri.info()
    assert (inst.n, inst.init_index, inst.goal_count) == (info["n"], info["init_index"], info["goal_count"])
    c, g, dev = inst.download()
    assert c.tobytes() == coords.tobytes()          # samples (with headings) bit for bit
    assert np.array_equal(dev.out_ptr, G.out_ptr) and np.array_equal(dev.out_col, G.out_col)
    assert dev.out_cost.tobytes() == G.out_cost.tobytes()
    # planning on the device-built graph (its own path points): the reference's result exactly
    want = ri.plan(spec.lam)
    assert want.status == abi.PLAN_SUCCESS
    assert not abi.full_parity(ctx.plan(inst, lam=spec.lam), want)
    ii = info["init_index"]
    assert not abi.full_parity(ctx.fmt_plan(inst, ii), ref.fmt_plan(spec, coords, len(gidx), G, ii))
    # and on the reference's own Dubins graph (cached paths) uploaded
    up = ctx.upload(spec, coords, len(gidx), G)
    assert not abi.full_parity(ctx.plan(up, ii, spec.lam, info["radius"]), want)
    assert not abi.full_parity(ctx.dijkstra_oracle(up, ii),
                               ref.dijkstra_oracle(spec, coords, len(gidx), G, ii))


@pytest.mark.parametrize("planar,rho,step", [(True, 0.05, 0.0), (False, 0.12, 0.004)])
def test_dubins_variants_plan_bitwise(ctx, ref, planar, rho, step):
    """3D Dubins airplane (climb), planar-cost-only (the hypot prune) and an
    explicit discretisation step: graph and plan exactly the reference's."""
    spec = forest_dubins()
    spec = P.extrude(spec, 3) if spec.dim == 2 else spec
    spec.steering, spec.init_heading, spec.radius_override = abi.STEER_DUBINS_AIRPLANE, 0.0, 0.3
    spec.dubins_rho, spec.dubins_step, spec.dubins_planar = rho, step, planar
    try:
        ri = ref.instance_build(spec)
    except Exception as e:  # (a scene the reference rejects is skipped)
        pytest.skip(str(e))
    coords, gidx, G = ri.graph(3)
    inst = ctx.build_instance(spec)
    c, g, dev = inst.download()
    assert c.tobytes() == coords.tobytes()
    assert np.array_equal(dev.out_col, G.out_col) and dev.out_cost.tobytes() == G.out_cost.tobytes()
    want = ri.plan(spec.lam)
    assert not abi.full_parity(ctx.plan(inst, lam=spec.lam), want)


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
    assert ob == tb  # the same file, byte for byte
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
