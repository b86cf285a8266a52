"""Device instance build times (warm, median of 3) for the configs' scenes."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_02403_b200 import native, problem as P  # noqa: E402

ctx = native.Context(0)
for name, spec in (("forest3d n=4000", P.forest_3d(3, 4000)), ("di6d n=4000", P.di_forest(3, 4000)),
                   ("quad12d n=8000", P.quad_scene())):
    ts = []
    for _ in range(4):
        t0 = time.perf_counter()
        inst = ctx.build_instance(spec)
        ctx.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
        e = inst.num_edges
        inst.close()
    print(f"{name}: build {statistics.median(ts[1:]):.1f} ms (first {ts[0]:.1f} ms), E={e}", flush=True)
