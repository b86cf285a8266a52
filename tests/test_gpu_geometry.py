"""Device exact geometry against the compiled reference: segment_free /
point_free (space.cpp:47-90) through the warp test every lazy check runs
(gmt_segment_free), on the reference's own KATs (tests/test_space.cpp:40-131)
and on a near-face corpus where the slab clip's starting values
tmin = 0, tmax = 1 (space.cpp:62-63) decide the outcome.  The bar is
bit-exact agreement on every segment."""
import numpy as np
import pytest

from paper_1705_02403_b200 import abi, problem as P
from paper_1705_02403_b200.graph import Graph

pytestmark = pytest.mark.gpu


def _spec(dim, lo, hi):
    lo = np.asarray(lo, np.float64).reshape(-1, dim)
    hi = np.asarray(hi, np.float64).reshape(-1, dim)
    return P.ProblemSpec(dim=dim, box_lo=lo, box_hi=hi, goal_lo=np.zeros(dim), goal_hi=np.ones(dim),
                         init=np.zeros(dim), n=10)


CENTER = ([0.4, 0.4], [0.6, 0.6])


@pytest.mark.parametrize("a,b,free", [
    # test_space.cpp:57-68 "segment_free basics"
    ([0.1, 0.1], [0.9, 0.9], False),
    ([0.1, 0.9], [0.9, 0.9], True),
    ([0.5, 0.5], [0.5, 0.5], False),
    ([0.3, 0.6], [0.7, 0.6], False),   # grazing a closed face is a hit
    # test_space.cpp:40-55 "point_free basics" as degenerate segments
    ([0.4, 0.5], [0.4, 0.5], False),   # box faces are blocked
    ([0.0, 0.0], [0.0, 0.0], True),    # the cube boundary is free
    ([1.0, 1.0], [1.0, 1.0], True),
    # the clip's parameter range: the line meets the box only beyond an end
    ([0.6 + 5e-10, 0.5], [0.9, 0.6], True),
    ([0.9, 0.6], [0.6 + 5e-10, 0.5], True),
    ([0.3, 0.4 - 1e-10], [0.1, 0.3], True),
    ([0.6 + 1e-12, 0.45], [0.95, 0.45], True),
    ([0.6, 0.45], [0.95, 0.45], False),  # starts on the face
])
def test_segment_kats(ctx, ref, a, b, free):
    spec = _spec(2, *CENTER)
    got = bool(ctx.segment_free(spec, [a], [b])[0])
    assert got == ref.segment_free(spec, a, b) == free


def test_segment_kats_no_boxes_and_planes(ctx, ref):
    empty = _spec(2, np.zeros((0, 2)), np.zeros((0, 2)))
    assert not ctx.segment_free(empty, [[0.5, 0.5]], [[1.5, 0.5]])[0]   # leaves the cube
    assert ctx.segment_free(empty, [[0.2, 0.2]], [[0.8, 0.3]])[0]
    plane = _spec(2, [0.5, 0.0], [0.5, 1.0])   # zero-thickness box: a blocking plane
    assert not ctx.segment_free(plane, [[0.5, 0.3]], [[0.5, 0.3]])[0]
    assert ctx.segment_free(plane, [[0.499, 0.3]], [[0.499, 0.3]])[0]
    assert not ctx.segment_free(plane, [[0.2, 0.3]], [[0.8, 0.3]])[0]
    assert ref.segment_free(plane, [0.499, 0.3], [0.499, 0.3])


def _random_boxes(rng, dim, count):
    # random_obstacles (test_space.cpp:23-36): lo ~ U[0, 0.8), hi = lo + U[0, 0.3)
    lo = rng.random((count, dim)) * 0.8
    return lo, lo + rng.random((count, dim)) * 0.3


def _near_face_corpus(rng, dim, lo, hi, m):
    """Segments with an endpoint 1e-12..1e-9 outside (or exactly on) a
    face of a random box, heading away from, along or into the box."""
    B = lo.shape[0]
    a = rng.random((m, dim))
    b = rng.random((m, dim))
    bi = rng.integers(0, B, m)
    ax = rng.integers(0, dim, m)
    side = rng.integers(0, 2, m)
    eps = 10.0 ** rng.uniform(-12, -9, m)
    eps[rng.random(m) < 0.05] = 0.0
    inside = rng.random(m) < 0.7           # other coordinates within the face's extent
    for i in range(m):
        k, j = ax[i], bi[i]
        if inside[i]:
            a[i] = lo[j] + rng.random(dim) * (hi[j] - lo[j])
        a[i, k] = (hi[j, k] + eps[i]) if side[i] else (lo[j, k] - eps[i])
        mode = rng.integers(0, 4)
        if mode == 0:      # away from the box along the face normal's side
            b[i, k] = a[i, k] + (1 if side[i] else -1) * rng.random() * 0.3
        elif mode == 1:    # parallel to the face
            b[i, k] = a[i, k]
        elif mode == 2:    # second endpoint also near a face of the same box
            b[i] = lo[j] + rng.random(dim) * (hi[j] - lo[j])
            kk = rng.integers(0, dim)
            b[i, kk] = (hi[j, kk] + eps[i]) if rng.integers(0, 2) else (lo[j, kk] - eps[i])
        # mode 3: b uniform
    swap = rng.random(m) < 0.5
    a[swap], b[swap] = b[swap].copy(), a[swap].copy()
    return np.clip(a, 0.0, 1.0), np.clip(b, 0.0, 1.0)


@pytest.mark.parametrize("dim,boxes", [(2, 3), (2, 40), (3, 12), (3, 60), (4, 8), (6, 20), (12, 6)])
def test_near_face_corpus_matches_reference(ctx, ref, dim, boxes):
    rng = np.random.default_rng(1000 + 7 * dim + boxes)
    lo, hi = _random_boxes(rng, dim, boxes)
    spec = _spec(dim, lo, hi)
    a, b = _near_face_corpus(rng, dim, lo, hi, 30000)
    want = ref.segment_free_many(spec, a, b).astype(bool)
    got = ctx.segment_free(spec, a, b)
    bad = np.flatnonzero(got != want)
    assert bad.size == 0, (f"{bad.size} of {len(a)} segments differ; first a={a[bad[0]].tolist()} "
                           f"b={b[bad[0]].tolist()} gpu={got[bad[0]]} ref={want[bad[0]]}")
    # the corpus exercises both outcomes
    assert 0.05 < want.mean() < 0.95


def test_symmetry_and_monotonicity(ctx, ref):
    """test_space.cpp:95-131: segment_free is symmetric, and adding a box
    never frees a blocked segment -- on the device and the reference."""
    rng = np.random.default_rng(1234)
    for rep in range(20):
        lo, hi = _random_boxes(rng, 2, 3)
        a, b = rng.random((500, 2)), rng.random((500, 2))
        spec = _spec(2, lo, hi)
        fwd = ctx.segment_free(spec, a, b)
        assert np.array_equal(fwd, ctx.segment_free(spec, b, a))
        assert np.array_equal(fwd, ref.segment_free_many(spec, a, b).astype(bool))
        lo2, hi2 = _random_boxes(rng, 2, 1)
        more = _spec(2, np.vstack([lo, lo2]), np.vstack([hi, hi2]))
        assert not np.any(ctx.segment_free(more, a, b) & ~fwd)


def test_two_node_plan_near_face(ctx, ref):
    """The near-face edge planned through the lazy check: box [0.4, 0.6]^2,
    init 5e-10 outside the right face, one goal sample up and to the right.
    The reference succeeds with cost 0.31622776554249626 along [1, 0]."""
    spec = P.ProblemSpec(dim=2, box_lo=np.array([[0.4, 0.4]]), box_hi=np.array([[0.6, 0.6]]),
                         goal_lo=np.array([0.85, 0.55]), goal_hi=np.array([0.95, 0.65]),
                         init=np.array([0.6 + 5e-10, 0.5]), n=1)
    coords = np.array([[0.9, 0.6], [0.6 + 5e-10, 0.5]])
    r = 0.5
    ptr, col, cost = ref.build_neighbor_graph(coords, r)
    g = Graph(2, r, ptr, col, cost, dim=2)
    want = ref.gmt_plan(spec, coords, 1, g, 1, 1.0, r)
    assert want.status == abi.PLAN_SUCCESS
    assert np.float64(want.cost).tobytes() == np.float64(0.31622776554249626).tobytes()
    assert want.path_indices.tolist() == [1, 0]
    inst = ctx.upload(spec, coords, 1, g)
    got = ctx.plan(inst, 1, 1.0, r)
    bad = abi.full_parity(got, want)
    assert not bad, f"mismatch in {bad}: gpu={got} ref={want}"
    fmt_g, fmt_r = ctx.fmt_plan(inst, 1), ref.fmt_plan(spec, coords, 1, g, 1)
    assert not abi.full_parity(fmt_g, fmt_r)
    dj_g = ctx.dijkstra_oracle(inst, 1)   # eager_check_kernel takes the same clip
    dj_r = ref.dijkstra_oracle(spec, coords, 1, g, 1)
    assert (dj_g.status, dj_g.cost, dj_g.total_collision_checks) == \
        (dj_r.status, dj_r.cost, dj_r.total_collision_checks)


def test_errors(ctx):
    from paper_1705_02403_b200.errors import InvalidInputError
    bad = _spec(2, [0.5, 0.5], [0.4, 0.6])   # lo > hi (validate_box, space.cpp:24-30)
    with pytest.raises(InvalidInputError):
        ctx.segment_free(bad, [[0.1, 0.1]], [[0.2, 0.2]])
