"""Probe C4 (12D quadrotor) parameters on the GPU: device build time,
edges, goal samples, plan status / cost / time for a grid of radii and
model scalings.  Usage: python tools/probe_quad.py"""
import itertools
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_1705_02403_b200 import native, problem as P  # noqa: E402


def main():
    ctx = native.Context()
    weights = [float(w) for w in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1.0, 0.3]
    radii = [float(r) for r in sys.argv[2].split(",")] if len(sys.argv) > 2 else [5.5, 6.0, 6.5]
    grid = [dict(vmax=0.5, amax=0.5, wmax=1.0, weight=w) for w in weights]
    for params, r in itertools.product(grid, radii):
        spec = P.quad_scene(5, 8000, radius=r)
        spec.quad_vmax, spec.quad_amax = params["vmax"], params["amax"]
        spec.quad_wmax, spec.quad_weight = params["wmax"], params["weight"]
        t0 = time.perf_counter()
        inst = ctx.build_instance(spec)
        t1 = time.perf_counter()
        res = ctx.plan(inst)
        t2 = time.perf_counter()
        times = []
        for _ in range(5):
            a = time.perf_counter()
            ctx.plan(inst)
            times.append(time.perf_counter() - a)
        print(f"{params} r={r} build {1e3 * (t1 - t0):.0f} ms E={inst.num_edges} "
              f"deg={inst.num_edges / inst.n:.1f} goals={inst.goal_count} status={res.status} "
              f"cost={res.cost:.3f} iters={res.iterations} checks={res.total_collision_checks} "
              f"plan {1e3 * np.median(times):.2f} ms", flush=True)


if __name__ == "__main__":
    main()
