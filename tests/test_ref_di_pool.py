"""The reference arm's double-integrator instances (bench.py --impl
reference): the reference's own sample_free + append_init, the graph from the
shared Halton pool rows re-indexed by rank plus direct rows of the non-pool
vertices.  They must equal the brute-force DI graph of the oracle's C
statement over the same samples (directed rows, costs, cached polylines), and
the unmodified reference planner must give the same plan on both."""
import numpy as np
import pytest

from paper_1705_02403_b200 import abi, problem as P
from helpers import bits


@pytest.mark.parametrize("q", [0, 1, 2])
def test_ref_di_pool_instance_equals_bruteforce(port, ref, q):
    spec = P.random_di_query(77, q, n=500, radius=2.3)
    pool = ref.di_pool(1, 2048, spec.di_params(), 2.3, 4)
    [ri] = ref.di_instances(pool, [spec], 2)
    coords, gidx, g = ri.graph(6)
    wc, wg = port.sample_free(spec)
    wc, wg, ii = port.append_init(wc, wg, spec.init, spec.goal_lo, spec.goal_hi)
    assert bits(coords) == bits(wc) and ri.info()["init_index"] == ii
    W = port.di_graph(wc, 2.3)
    assert np.array_equal(g.out_ptr, W.out_ptr) and np.array_equal(g.out_col, W.out_col)
    assert bits(g.out_cost) == bits(W.out_cost)
    assert np.array_equal(g.in_ptr, W.in_ptr) and np.array_equal(g.in_col, W.in_col)
    assert bits(g.in_cost) == bits(W.in_cost)
    assert bits(g.path_pts) == bits(W.path_pts)
    for lam in (1.0, 0.5):
        got = ri.plan(lam)
        want = ref.gmt_plan(spec, wc, len(wg), W, ii, lam, 2.3)
        assert not abi.full_parity(got, want)
