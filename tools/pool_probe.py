"""Timing probe of the configs[4] pipeline: 4096 random 6D double-integrator
queries (n=4000, r=1.6) through the shared Halton pool."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1705_02403_b200 import abi, problem as P
from paper_1705_02403_b200.native import Context, ProblemBatch

Q = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
ctx = Context(0)
t0 = time.perf_counter()
specs = [P.random_di_query(20171005, q, n=4000, radius=1.6) for q in range(Q)]
pb = ProblemBatch(specs)
print(f"specs {time.perf_counter()-t0:.2f}s", flush=True)
for it in range(3):
    t0 = time.perf_counter()
    st, summ, _ = ctx.plan_problems(pb)
    dt = time.perf_counter() - t0
    print(f"plan_problems {dt*1e3:.1f} ms  ({Q/dt:.0f} plans/s)  ok={int((st==0).sum())} "
          f"success={sum(1 for s in summ if s.status==0)} pool={ctx.pool_info()}", flush=True)
t0 = time.perf_counter()
b, st = ctx.batch_problems(pb)
ctx.synchronize()
print(f"batch_problems {1e3*(time.perf_counter()-t0):.1f} ms", flush=True)
stream = torch.cuda.ExternalStream(ctx.stream)
for it in range(2):
    b.launch()
ctx.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for it in range(5):
    b.launch()
e1.record(stream)
e1.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"solve launch {ms:.2f} ms -> {Q/ms*1e3:.0f} plans/s device-resident", flush=True)
s2 = b.summaries()
assert [(a.status, a.cost) for a in s2] == [(a.status, a.cost) for a, s in zip(summ, st) if s == 0]
os.environ["GMT_POOL_TIMING"] = "1"
for it in range(2):
    t0 = time.perf_counter()
    st, summ, _ = ctx.plan_problems(pb)
    dt = time.perf_counter() - t0
    print(f"timed plan_problems {dt*1e3:.1f} ms stages={['%.2f' % x for x in ctx.pool_info()['stage_ms']]} "
          f"fallbacks={ctx.pool_info()['last_fallbacks']}", flush=True)
