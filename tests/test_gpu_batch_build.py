"""GPU: the batched build_instance + gmt_plan (gmt_plan_problems) equals
gmt_instance_build + gmt_plan problem by problem -- statuses, costs,
iterations, checks and the path states -- including the problems that take
sample_free's rare paths (goal substitution, goal blocked, exhausted
budget), uniform and Halton sampling, and the reference on a sample."""
import numpy as np
import pytest

from paper_1705_02403_b200 import abi, problem as P
from paper_1705_02403_b200.errors import GoalBlockedError, InfeasibleSamplingError
from helpers import scene

pytestmark = pytest.mark.gpu


def _mixed_specs():
    specs = [P.random_forest_query(20171005, q, n=1500) for q in range(24)]
    for seed in (3, 9, 27):
        u = scene("rectangles_2d", 400)
        u.sampling_kind, u.seed = abi.SAMPLE_UNIFORM, seed
        specs.append(u)
    tiny = scene("rectangles_2d", 300)  # goal too small for any sample: substitution
    tiny.goal_lo, tiny.goal_hi = np.array([0.95, 0.30]), np.array([0.9501, 0.3001])
    specs.append(tiny)
    blocked = scene("rectangles_2d", 300)  # goal inside an obstacle: GoalBlockedError
    blocked.goal_lo, blocked.goal_hi = np.array([0.25, 0.1]), np.array([0.3, 0.2])
    specs.append(blocked)
    crowded = scene("rectangles_2d", 200)  # nearly all space blocked: more than the first chunk
    crowded.box_lo = np.vstack([crowded.box_lo, [[0.0, 0.0]]])
    crowded.box_hi = np.vstack([crowded.box_hi, [[1.0, 0.97]]])
    crowded.init = np.array([0.05, 0.99])
    crowded.goal_lo, crowded.goal_hi = np.array([0.9, 0.98]), np.array([1.0, 1.0])
    specs.append(crowded)
    specs.append(scene("maze_3d", 800).with_n(800) if False else P.forest_3d(3, 900))
    return specs


def test_plan_problems_matches_single_builds(ctx):
    specs = [s for s in _mixed_specs() if s.dim == 3][:20]
    specs2 = [s for s in _mixed_specs() if s.dim == 2]
    for group in (specs, specs2):
        cap = 4096
        status, summ, paths = ctx.plan_problems(group, path_cap=cap)
        for q, sp in enumerate(group):
            try:
                inst = ctx.build_instance(sp)
            except GoalBlockedError:
                assert status[q] == 3
                continue
            except InfeasibleSamplingError:
                assert status[q] == 2
                continue
            assert status[q] == 0
            want = ctx.plan(inst, lam=sp.lam)
            got = summ[q]
            assert (got.status, got.iterations, got.total_collision_checks, got.path_len) == (
                want.status, want.iterations, want.total_collision_checks, len(want.path_indices))
            assert got.cost == want.cost or (np.isinf(got.cost) and np.isinf(want.cost))
            if want.status == abi.PLAN_SUCCESS:
                c, _, _ = inst.download()
                assert paths[q, :got.path_len].tobytes() == c[want.path_indices].tobytes()


def test_plan_problems_matches_reference(ctx, ref):
    specs = [P.random_forest_query(7, q, n=1200) for q in range(6)]
    status, summ, _ = ctx.plan_problems(specs)
    for q, sp in enumerate(specs):
        want = ref.instance_build(sp).plan(sp.lam)
        assert status[q] == 0
        assert (summ[q].status, summ[q].cost, summ[q].iterations, summ[q].total_collision_checks) == (
            want.status, want.cost, want.iterations, want.total_collision_checks)


def test_plan_problems_generic_dimension_and_errors(ctx):
    """d = 6 takes the generic r-disk kernel (no row scratch); a batch mixing
    Euclidean and double-integrator problems, and mixed dimensions, are
    rejected (double-integrator batches take the shared pool,
    tests/test_gpu_pool.py)."""
    specs = [scene("rectangles_6d", 400 + 50 * k) for k in range(4)]
    status, summ, _ = ctx.plan_problems(specs)
    for q, sp in enumerate(specs):
        want = ctx.plan(ctx.build_instance(sp), lam=sp.lam)
        assert status[q] == 0
        assert (summ[q].status, summ[q].cost, summ[q].iterations) == (want.status, want.cost, want.iterations)
    from paper_1705_02403_b200.errors import InvalidInputError
    with pytest.raises(InvalidInputError):
        ctx.plan_problems([scene("rectangles_6d", 300), P.di_forest(3, 300)])
    di = P.di_forest(3, 300, radius=2.6)
    status, summ, _ = ctx.plan_problems([di])
    want = ctx.plan(ctx.build_instance(di))
    assert status[0] == 0 and (summ[0].status, summ[0].cost) == (want.status, want.cost)
    with pytest.raises(InvalidInputError):
        ctx.plan_problems([scene("rectangles_2d", 200), scene("rectangles_3d", 200)])


def test_plan_problems_rdisk_grid_equals_brute_scan(ctx, monkeypatch):
    """The grid-binned r-disk pass (d = 2, 3) against the all-pairs scan
    (GMT_NO_RDISK_GRID): summaries and paths bit for bit, over radii from
    one cell (G = 1) to the cell cap, and sizes past the grid's row limit
    (which take the scan)."""
    import dataclasses
    specs = [P.random_forest_query(11, q, n=4000) for q in range(6)]
    specs += [dataclasses.replace(P.random_forest_query(12, q, n=2500), radius_override=r)
              for q, r in enumerate((0.9, 0.3, 0.05, 0.02))]
    specs2 = [scene("rectangles_2d", n) for n in (300, 2000, 6000)]
    specs2 += [dataclasses.replace(scene("rectangles_2d", 3000), radius_override=r) for r in (1.5, 0.004)]
    big = [P.random_forest_query(13, q, n=9000) for q in range(2)]
    for group in (specs, specs2, big):
        cap = 2048
        got = ctx.plan_problems(group, path_cap=cap)  # grid rows, solved in place (row-padded) when none overflows
        monkeypatch.setenv("GMT_BATCH_CSR", "1")
        csr = ctx.plan_problems(group, path_cap=cap)  # grid rows compacted into a CSR
        monkeypatch.setenv("GMT_NO_RDISK_GRID", "1")
        want = ctx.plan_problems(group, path_cap=cap)  # all-pairs rows, CSR
        monkeypatch.delenv("GMT_NO_RDISK_GRID")
        monkeypatch.delenv("GMT_BATCH_CSR")
        for other in (got, csr):
            assert other[0].tolist() == want[0].tolist()
            for a, b in zip(other[1], want[1]):
                assert (a.status, a.iterations, a.total_collision_checks, a.path_len) == (
                    b.status, b.iterations, b.total_collision_checks, b.path_len)
                assert a.cost == b.cost or (np.isinf(a.cost) and np.isinf(b.cost))
            assert other[2].tobytes() == want[2].tobytes()


def test_plan_problems_concurrent_contexts_and_scratch_reuse(ctx):
    """Reentrancy (simulator.cpp:212 plans from several threads): two
    contexts calling gmt_plan_problems from two host threads, with batches
    of different sizes so each context's kept scratch is reused, grown and
    reused again, give exactly the one-thread results."""
    import threading
    from paper_1705_02403_b200 import native
    groups = [[P.random_forest_query(11, q, n=1000 + 250 * (k % 2)) for q in range(8 + 8 * k)] for k in range(4)]
    want = [ctx.plan_problems(g, path_cap=256) for g in groups]
    ctxs = [ctx, native.Context(0)]
    got = [[None] * len(groups) for _ in ctxs]

    def work(i):
        order = range(len(groups)) if i == 0 else reversed(range(len(groups)))
        for _ in range(2):
            for k in order:
                got[i][k] = ctxs[i].plan_problems(groups[k], path_cap=256)

    try:
        th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
        for t in th:
            t.start()
        for t in th:
            t.join()
    finally:
        ctxs[1].close()
    for i in range(2):
        for k, (ws, wsum, wp) in enumerate(want):
            gs, gsum, gp = got[i][k]
            assert list(gs) == list(ws)
            assert [(a.status, a.cost, a.iterations, a.total_collision_checks, a.path_len) for a in gsum] == \
                [(b.status, b.cost, b.iterations, b.total_collision_checks, b.path_len) for b in wsum]
            assert gp.tobytes() == wp.tobytes()
