"""GPU parity against the unmodified reference planner at the sizes
BASELINE.json names (configs[1-4]), not only on small instances:

* configs[2]: the 6D double integrator di_forest(3, 4000), r = 1.6,
  lambda in {1, 0.5} -- device instance (samples, DI graph, solve with the
  trajectories regenerated in the kernel) vs the reference gmt_plan on the
  reference's own samples with the DI graph and cached polylines of the
  oracle's model statement (built over the shared Halton pool,
  tests/test_ref_di_pool.py pins that construction to brute force);
* configs[3]: the 12D quadrotor quad_scene() at n = 8000 -- the device graph
  with its waypoint polylines injected into the reference gmt_plan, the
  graph spot-checked pair by pair against the oracle's model statement;
* configs[1]: 32 random 3D forest queries at n = 4000 through
  gmt_plan_problems vs the reference build_instance + gmt_plan;
* configs[4]: 64 batched random DI queries (n = 4000, r = 1.6) through the
  shared-pool gmt_plan_problems vs the reference.
The bar is the reference's bitwise same_tree plus iterations, checks and
per-pass stats (full trees), or status / cost bits / iterations / checks
(batched summaries)."""
import os

import numpy as np
import pytest

from paper_1705_02403_b200 import abi, problem as P
from helpers import bits

pytestmark = pytest.mark.gpu

THREADS = min(os.cpu_count() or 1, 32)


def _summary_key(s):
    return (s.status, np.float64(s.cost).tobytes(), s.iterations, s.total_collision_checks)


@pytest.fixture(scope="module")
def di4000(ctx, ref):
    spec = P.di_forest(3, 4000, radius=1.6)
    pool = ref.di_pool(spec.start_index, P.halton_pool_size([spec]), spec.di_params(), 1.6, THREADS)
    [ri] = ref.di_instances(pool, [spec], 1)
    return spec, ri, ctx.build_instance(spec)


def test_di_n4000_graph_matches_oracle_statement(di4000):
    spec, ri, inst = di4000
    wc, _, g = ri.graph(6)
    coords, gidx, G = inst.download()
    assert bits(coords) == bits(wc)
    assert inst.init_index == ri.info()["init_index"]
    assert np.array_equal(G.out_ptr, g.out_ptr) and np.array_equal(G.out_col, g.out_col)
    assert bits(G.out_cost) == bits(g.out_cost)
    assert G.num_edges > 100000   # ~34 out-edges per vertex at r = 1.6


@pytest.mark.parametrize("lam", [1.0, 0.5])
def test_di_n4000_plan_matches_reference(ctx, di4000, lam):
    spec, ri, inst = di4000
    want = ri.plan(lam)
    got = ctx.plan(inst, lam=lam)
    assert want.status == abi.PLAN_SUCCESS
    assert not abi.full_parity(got, want), abi.full_parity(got, want)


def test_quad_n8000_plan_matches_reference(ctx, port, ref):
    spec = P.quad_scene()
    inst = ctx.build_instance(spec)
    coords, gidx, _ = inst.download()
    ii = inst.init_index
    qp = spec.quad_params()
    G = ctx.build_quad_graph(coords, qp, spec.radius_override, paths=True)
    assert G.num_edges > 400000
    # the graph against the oracle's statement of the model: every out-edge of
    # 24 vertices and 3000 random pairs (cost <= r exactly where an edge is)
    rng = np.random.default_rng(8000)
    for u in rng.choice(G.n, 24, replace=False):
        a, b = G.out_ptr[u], G.out_ptr[u + 1]
        for v, c in zip(G.out_col[a:b], G.out_cost[a:b]):
            wc, _ = port.quad_cost(coords[u], coords[v], qp)
            assert np.float64(wc).tobytes() == np.float64(c).tobytes()
    for u, v in rng.integers(0, G.n, (3000, 2)):
        if u == v:
            continue
        wc, _ = port.quad_cost(coords[u], coords[v], qp)
        a, b = G.out_ptr[u], G.out_ptr[u + 1]
        assert (wc <= spec.radius_override) == bool(np.any(G.out_col[a:b] == v))
    want = ref.gmt_plan(spec, coords, len(gidx), G, ii, 1.0, spec.radius_override)
    got = ctx.plan(inst)
    assert want.status == abi.PLAN_SUCCESS
    assert not abi.full_parity(got, want), abi.full_parity(got, want)


def test_forest_n4000_batch_matches_reference(ctx, ref):
    specs = [P.random_forest_query(20171005, q, n=4000) for q in range(32)]
    insts = ref.instance_build_many(specs, THREADS)
    want, _ = ref.plan_many(insts, 1.0, THREADS)
    status, got, _ = ctx.plan_problems(specs)
    assert (status == 0).all()
    assert [_summary_key(s) for s in got] == [_summary_key(s) for s in want]
    for q in (0, 7, 31):  # full trees
        d = ctx.plan(ctx.build_instance(specs[q]))
        assert not abi.full_parity(d, insts[q].plan(1.0))


def test_di_batched_configs4_matches_reference(ctx, ref):
    specs = [P.random_di_query(20171005, q, n=4000, radius=1.6) for q in range(64)]
    pool = ref.di_pool(1, P.halton_pool_size(specs), specs[0].di_params(), 1.6, THREADS)
    insts = ref.di_instances(pool, specs, THREADS)
    want, _ = ref.plan_many(insts, 1.0, THREADS)
    status, got, _ = ctx.plan_problems(specs)
    assert (status == 0).all()
    assert [_summary_key(s) for s in got] == [_summary_key(s) for s in want]
    b, st = ctx.batch_problems(specs[:8])
    b.launch()
    for q in range(8):  # full trees of the derived instances
        assert not abi.full_parity(b.result(q), insts[q].plan(1.0))
