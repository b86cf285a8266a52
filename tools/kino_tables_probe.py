"""Single-solve p50 (16-CTA cluster) of configs[2] (DI n = 4000) and
configs[3] (quadrotor n = 8000) with the build-time waypoint tables on and
off (GMT_KINO_TABLES), plus bitwise equality of the two plans."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1705_02403_b200 import abi, problem as P  # noqa: E402
from paper_1705_02403_b200.native import OPT_BATCH_CLUSTER, OPT_BATCH_THREADS, Context  # noqa: E402

ctx = Context(0)
stream = torch.cuda.ExternalStream(ctx.stream_handle()) if hasattr(ctx, "stream_handle") else None


def p50(inst, reps=51):
    ctx.set_option(OPT_BATCH_CLUSTER, 16)
    ctx.set_option(OPT_BATCH_THREADS, 0)
    b = ctx.batch([inst], 1.0)
    ctx.set_option(OPT_BATCH_CLUSTER, 0)
    for _ in range(5):
        b.launch()
    ctx.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        b.launch()
        ctx.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    b.close()
    return statistics.median(ts)


for name, spec in (("di n=4000", P.di_forest(3, 4000)), ("quad n=8000", P.quad_scene())):
    res = {}
    for mode in ("0", "1"):
        os.environ["GMT_KINO_TABLES"] = mode
        t0 = time.perf_counter()
        inst = ctx.build_instance(spec)
        ctx.synchronize()
        build = (time.perf_counter() - t0) * 1e3
        r = ctx.plan(inst)
        res[mode] = r
        print(f"{name} tables={mode}: build {build:.1f} ms, p50 {p50(inst):.3f} ms (host clock), "
              f"status {r.status} iters {r.iterations} checks {r.total_collision_checks}", flush=True)
        del inst
    print(name, "plans identical:", not abi.full_parity(res["0"], res["1"]))
