"""Dubins on the device vs the reference: cost agreement statistics and the
forest_dubins instance / plan comparison (numbers quoted in DESIGN.md §3.4)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1705_02403_b200 import abi, native  # noqa: E402
from test_gpu_dubins import _params, forest_dubins  # noqa: E402

ctx, ref = native.Context(0), oracle.ref()
for dim, planar in ((2, False), (3, False)):
    rng = np.random.default_rng(5)
    m = 100000
    x0, x1 = rng.random((m, dim + 1)), rng.random((m, dim + 1))
    x0[:, dim] *= 2 * np.pi
    x1[:, dim] *= 2 * np.pi
    p = _params(0.08, 0.0, planar)
    c, s = ctx.dubins_costs(x0, x1, dim, p)
    rc, rs = ref.dubins_costs(x0, x1, dim, p)
    ulps = np.abs(c.view(np.int64) - rc.view(np.int64))
    print(f"dim {dim}: {m} pairs, bit-identical costs {np.mean(c == rc):.4f}, max |ulp diff| {ulps.max()}, "
          f"max rel {np.max(np.abs(c - rc) / rc):.2e}, segment counts equal {np.mean(s == rs):.5f}")
spec = forest_dubins()
ri = ref.instance_build(spec)
coords, gidx, G = ri.graph(2)
inst = ctx.build_instance(spec)
c, g, dev = inst.download()
same_edges = np.array_equal(dev.out_ptr, G.out_ptr) and np.array_equal(dev.out_col, G.out_col)
print(f"forest_dubins: n={inst.n} E={inst.num_edges} (ref {G.num_edges}) same edge set {same_edges}, "
      f"bit-identical edge costs {np.mean(dev.out_cost == G.out_cost) if same_edges else float('nan'):.4f}")
want, got = ri.plan(spec.lam), ctx.plan(inst, lam=spec.lam)
print(f"plan: ref status {want.status} cost {want.cost!r} iters {want.iterations} checks {want.total_collision_checks}; "
      f"device {got.status} {got.cost!r} {got.iterations} {got.total_collision_checks}; "
      f"full parity mismatches on the device-built graph: {abi.full_parity(got, want)}")
