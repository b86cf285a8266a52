"""Batched double-integrator queries over the shared Halton sample pool
(SURVEY.md §8(e), configs[4]): every derived per-query graph equals the graph
gmt_instance_build builds for that problem alone, bit for bit (coordinates,
in-rows with costs and durations, out-rows), and the batched solves equal the
per-instance solves -- full trees, stats and summaries.  The per-instance
path is itself pinned to the oracle's DI statement and to the unmodified
reference planner (tests/test_gpu_di.py, tests/test_gpu_fullsize.py)."""
import numpy as np
import pytest

from paper_1705_02403_b200 import abi, problem as P
from helpers import bits

pytestmark = pytest.mark.gpu

MASTER = 20171005


def _same_graph(a, b):
    assert a["n"] == b["n"]
    V = a["n"]
    assert bits(a["coords"][: V * 6]) == bits(b["coords"][: V * 6]), "coords"
    assert np.array_equal(a["in_ptr"], b["in_ptr"]), "in_ptr"
    assert np.array_equal(a["in_col"], b["in_col"]), "in_col"
    assert bits(a["in_cost"]) == bits(b["in_cost"]), "in_cost"
    assert bits(a["in_tau"]) == bits(b["in_tau"]), "in_tau"
    assert np.array_equal(a["out_ptr"], b["out_ptr"]), "out_ptr"
    assert np.array_equal(a["out_col"], b["out_col"]), "out_col"


def _halton(index, base):
    """radical inverse (sampling.cpp:21-34), the same IEEE steps."""
    f, r = 1.0, 0.0
    while index > 0:
        f /= base
        r += f * (index % base)
        index //= base
    return r


def _specs(count, n=4000, radius=1.6, master=MASTER, first=0):
    return [P.random_di_query(master, q, n=n, radius=radius) for q in range(first, first + count)]


@pytest.fixture(scope="module")
def full64(ctx):
    specs = _specs(64)
    pb, status = ctx.batch_problems(specs)
    assert (status == 0).all()
    insts = [ctx.build_instance(s) for s in specs]
    ib = ctx.batch(insts, 1.0)
    return specs, pb, ib, insts


def test_pool_graphs_equal_single_builds(ctx, full64):
    specs, pb, ib, _ = full64
    for q in range(len(specs)):
        _same_graph(pb.graph(q), ib.graph(q))
    assert ctx.pool_info()["pool_size"] >= 4000


def test_pool_batch_results_equal_single_builds(ctx, full64):
    specs, pb, ib, _ = full64
    pb.launch()
    ib.launch()
    sa, sb = pb.summaries(), ib.summaries()
    for q in range(len(specs)):
        assert (sa[q].status, sa[q].cost, sa[q].iterations, sa[q].total_collision_checks, sa[q].path_len) == \
            (sb[q].status, sb[q].cost, sb[q].iterations, sb[q].total_collision_checks, sb[q].path_len), q
    for q in range(0, len(specs), 7):
        bad = abi.full_parity(pb.result(q), ib.result(q))
        assert not bad, (q, bad)
    assert sum(1 for s in sa if s.status == abi.PLAN_SUCCESS) > len(specs) // 2


def test_plan_problems_di_matches_batches(ctx, full64):
    specs, pb, _, insts = full64
    status, summ, paths = ctx.plan_problems(specs, path_cap=64)
    assert (status == 0).all()
    pb.launch()
    ref = pb.summaries()
    for q, (a, b) in enumerate(zip(summ, ref)):
        assert (a.status, a.cost, a.iterations, a.total_collision_checks) == \
            (b.status, b.cost, b.iterations, b.total_collision_checks), q
    # path states: the plan's vertices' coordinates
    for q in range(0, len(specs), 9):
        if summ[q].status != abi.PLAN_SUCCESS:
            continue
        r = ctx.plan(insts[q])
        c, _, _ = insts[q].download()
        L = min(len(r.path_indices), 64)
        want = c[r.path_indices[:L]]
        assert bits(paths[q, :L]) == bits(np.ascontiguousarray(want))


@pytest.mark.parametrize("lam", [0.5, 0.2])
def test_pool_lambda(ctx, lam):
    specs = _specs(16, first=100)
    for s in specs:
        s.lam = lam
    status, summ, _ = ctx.plan_problems(specs)
    assert (status == 0).all()
    for s, a in zip(specs, summ):
        r = ctx.plan(ctx.build_instance(s), lam=lam)
        assert (a.status, a.cost, a.iterations, a.total_collision_checks) == \
            (r.status, r.cost, r.iterations, r.total_collision_checks)


def test_pool_rare_paths(ctx):
    """Off the fast path, each problem still equals its single build: an init
    that duplicates a sample exactly (append_init reuses the index), a scene
    whose goal centre is blocked (the Halton search of sampling.cpp:120-141),
    a problem too dense for the pool estimate, and a small-n query."""
    specs = _specs(6, n=800, radius=2.2, first=500)
    # (0) init = the query's first free Halton sample
    port_pts = np.array([[_halton(i, p) for p in (2, 3, 5, 7, 11, 13)] for i in range(1, 50)])
    s0 = specs[0]
    for pt in port_pts:
        if s0.point_free(pt):
            s0.init = pt.copy()
            break
    # (1) a box over the goal centre
    s1 = specs[1]
    gc = 0.5 * (s1.goal_lo + s1.goal_hi)
    lo = gc - 0.004
    hi = gc + 0.004
    lo[3:], hi[3:] = 0.0, 1.0
    s1.box_lo = np.vstack([s1.box_lo, lo])
    s1.box_hi = np.vstack([s1.box_hi, hi])
    # (2) a slab over most of x: the free-volume estimate sizes the pool too
    # small for this query (it then takes the single builder)
    s2 = specs[2]
    s2.box_lo = np.vstack([s2.box_lo, [0.1, 0.0, 0.0, 0.0, 0.0, 0.0]])
    s2.box_hi = np.vstack([s2.box_hi, [0.88, 1.0, 1.0, 1.0, 1.0, 1.0]])
    specs[3] = P.random_di_query(MASTER, 503, n=2, radius=2.2)
    status, summ, _ = ctx.plan_problems(specs)
    pb, st2 = ctx.batch_problems(specs)
    assert np.array_equal(status, st2)
    k = 0
    for q, s in enumerate(specs):
        if status[q] != 0:
            continue
        inst = ctx.build_instance(s)
        r = ctx.plan(inst)
        assert (summ[q].status, summ[q].cost, summ[q].iterations) == (r.status, r.cost, r.iterations), q
        _same_graph(pb.graph(k), ctx.batch([inst], 1.0).graph(0))
        k += 1


def test_pool_views_equal_materialised_rows(ctx, monkeypatch):
    """gmt_plan_problems reads each query's graph through its rank map over
    the pool rows; device-resident batches materialise every derived row
    (GMT_POOL_ROWS=0/1 forces either).  Both give the same graphs and the
    same full results, and plan_problems the same summaries either way."""
    specs = _specs(24, first=300)
    monkeypatch.setenv("GMT_POOL_ROWS", "0")
    pv, _ = ctx.batch_problems(specs)
    sv = ctx.plan_problems(specs)[1]
    monkeypatch.setenv("GMT_POOL_ROWS", "1")
    pm, _ = ctx.batch_problems(specs)
    sm = ctx.plan_problems(specs)[1]
    monkeypatch.delenv("GMT_POOL_ROWS")
    assert [(a.status, a.cost, a.iterations) for a in sv] == [(a.status, a.cost, a.iterations) for a in sm]
    pv.launch()
    pm.launch()
    for q in range(len(specs)):
        _same_graph(pv.graph(q), pm.graph(q))
        assert not abi.full_parity(pv.result(q), pm.result(q))


def test_pool_check_records_equal_regeneration(ctx, monkeypatch):
    """The pool's per-edge check records (bounding box, cube test and the
    waypoint positions of each pool edge, built once with the pool graph)
    replace the lazy check's table regeneration on pool edges: the same
    results, full trees included, with GMT_POOL_REC=0 (a fresh context's pool
    without records) as with them, through views and materialised rows."""
    from paper_1705_02403_b200.native import Context
    specs = _specs(96, first=500)
    on_st, on_s, _ = ctx.plan_problems(specs)
    on_b, _ = ctx.batch_problems(specs[:16])
    on_b.launch()
    monkeypatch.setenv("GMT_POOL_REC", "0")
    off = Context(0)
    off_st, off_s, _ = off.plan_problems(specs)
    off_b, _ = off.batch_problems(specs[:16])
    off_b.launch()
    monkeypatch.delenv("GMT_POOL_REC")
    assert (on_st == 0).all() and (off_st == 0).all()
    key = lambda s: (s.status, bits([s.cost]), s.iterations, s.total_collision_checks)  # noqa: E731
    assert [key(s) for s in on_s] == [key(s) for s in off_s]
    for q in range(16):
        assert not abi.full_parity(on_b.result(q), off_b.result(q)), q


def test_pool_smaller_queries_after_larger():
    """A context's pool grows to the largest query it has seen; a later call
    with smaller queries scans fewer pool points (its rank maps are shorter
    than the pool graph), yet pool rows still name every pool point: those
    past the scan are no query's vertices.  Graphs and results equal the
    single builds."""
    from paper_1705_02403_b200.native import Context
    c = Context(0)
    big = _specs(8, n=4000, first=700)
    st, _, _ = c.plan_problems(big)
    assert (st == 0).all()
    small = _specs(16, n=900, first=720)
    st, summ, _ = c.plan_problems(small)
    pb, st2 = c.batch_problems(small)
    assert (st == 0).all() and (st2 == 0).all()
    pb.launch()
    for q, s in enumerate(small):
        inst = c.build_instance(s)
        r = c.plan(inst)
        assert (summ[q].status, summ[q].cost, summ[q].iterations, summ[q].total_collision_checks) == \
            (r.status, r.cost, r.iterations, r.total_collision_checks), q
        _same_graph(pb.graph(q), c.batch([inst], 1.0).graph(0))
        assert not abi.full_parity(pb.result(q), r), q
