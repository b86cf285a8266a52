"""Queries above the shared-memory wavefront limit (about 18k vertices):
the solve keeps its wavefront state in a per-query global buffer (one wide
CTA per query, SolveJob::gstate) instead of failing.  The reference planner
has no size limit (planner.cpp:94-198); these compare with it at n = 30000
(2D) and 25000 (3D) -- single solves, fmt_plan, batches and the batched
offline path -- bit for bit."""
import numpy as np
import pytest

from paper_1705_02403_b200 import abi, problem as P
from helpers import scene

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def big2d(ctx, ref):
    spec = scene("rectangles_2d", 30000)
    return spec, ref.instance_build(spec), ctx.build_instance(spec)


@pytest.mark.parametrize("lam", [1.0, 0.5])
def test_n30000_plan_matches_reference(ctx, big2d, lam):
    spec, ri, inst = big2d
    assert inst.n == 30001
    want = ri.plan(lam)
    got = ctx.plan(inst, lam=lam)
    assert want.status == abi.PLAN_SUCCESS
    assert not abi.full_parity(got, want), abi.full_parity(got, want)


def test_n30000_fmt_and_batch(ctx, ref, big2d):
    spec, ri, inst = big2d
    b = ctx.batch([inst, inst], 1.0)
    b.launch()
    want = ri.plan(1.0)
    for q in range(2):
        assert not abi.full_parity(b.result(q), want)
    c, gi, G = inst.download()
    fmt = ctx.fmt_plan(inst)
    assert not abi.full_parity(fmt, ref.fmt_plan(spec, c, len(gi), G, inst.init_index))


def test_large_batched_problems_match_reference(ctx, ref):
    specs = [P.random_forest_query(99, q, n=25000) for q in range(2)] + \
            [P.random_forest_query(99, 2, n=3000)]  # mixed: on-chip and global state in one batch
    status, summ, _ = ctx.plan_problems(specs)
    insts = ref.instance_build_many(specs, 4)
    want, _ = ref.plan_many(insts, 1.0, 4)
    assert (status == 0).all()
    for a, b in zip(summ, want):
        assert (a.status, np.float64(a.cost).tobytes(), a.iterations, a.total_collision_checks) == \
            (b.status, np.float64(b.cost).tobytes(), b.iterations, b.total_collision_checks)


def test_above_u16_ids_matches_reference(ctx, ref):
    """n = 70000 (> 65535, past the on-chip u16 vertex ids): the global
    wavefront uses 32-bit work lists."""
    spec = scene("rectangles_2d", 70000)
    ri = ref.instance_build(spec)
    inst = ctx.build_instance(spec)
    assert inst.n == 70001
    got, want = ctx.plan(inst), ri.plan(1.0)
    assert want.status == abi.PLAN_SUCCESS
    assert not abi.full_parity(got, want), abi.full_parity(got, want)
