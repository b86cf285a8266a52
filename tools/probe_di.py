"""C3 probe: 6D double integrator, n=4000 -- build time, single-solve p50, batched rate."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1705_02403_b200 import problem as P  # noqa: E402
from paper_1705_02403_b200.native import Context, OPT_BATCH_CLUSTER, OPT_BATCH_THREADS  # noqa: E402

ctx = Context(0)
stream = torch.cuda.ExternalStream(ctx.stream)
spec = P.di_forest(3, 4000)
t0 = time.perf_counter()
inst = ctx.build_instance(spec)
ctx.synchronize()
print(f"build (sample+append+DI graph) {1e3 * (time.perf_counter() - t0):.1f} ms, E={inst.num_edges}, "
      f"deg={inst.num_edges / inst.n:.1f}")
r = ctx.plan(inst)
print("plan:", r, "passes", len(r.group_sizes))
for cs in (8, 16):
    ctx.set_option(OPT_BATCH_CLUSTER, cs)
    ctx.set_option(OPT_BATCH_THREADS, 0)
    b = ctx.batch([inst], 1.0)
    ctx.set_option(OPT_BATCH_CLUSTER, 0)
    for _ in range(5):
        b.launch()
    ctx.synchronize()
    ts = []
    for _ in range(51):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        b.launch()
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"cluster {cs}: p50 {statistics.median(ts):.3f} ms")
Q = int(sys.argv[1]) if len(sys.argv) > 1 else 128
t0 = time.perf_counter()
insts = [ctx.build_instance(P.random_di_query(20171005, q, n=4000)) for q in range(Q)]
print(f"built {Q} DI queries in {time.perf_counter() - t0:.1f} s")
for cs, thr in ((1, 256), (2, 0)):
    ctx.set_option(OPT_BATCH_CLUSTER, cs)
    ctx.set_option(OPT_BATCH_THREADS, thr)
    b = ctx.batch(insts, 1.0)
    for _ in range(3):
        b.launch()
    ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(5):
        b.launch()
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 5
    s = b.summaries()
    print(f"batch cs={cs}: {ms:.2f} ms per {Q} -> {Q / ms * 1e3:.0f} plans/s; "
          f"solved {sum(1 for x in s if x.status == 0)}/{Q}")
