"""Problems -> plans throughput: gmt_plan_problems (batched offline phase +
one batched solve) vs one gmt_instance_build per problem + a batched solve."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1705_02403_b200 import native, problem as P  # noqa: E402

q = int(sys.argv[1]) if len(sys.argv) > 1 else 512
ctx = native.Context(0)
specs = [P.random_forest_query(20171005, i, n=4000) for i in range(q)]
for rep in range(3):
    t0 = time.perf_counter()
    status, summ, _ = ctx.plan_problems(specs)
    t1 = time.perf_counter()
print(f"gmt_plan_problems: {q} problems in {1e3 * (t1 - t0):.1f} ms -> {q / (t1 - t0):.0f} plans/s "
      f"(solved {sum(1 for s in summ if s.status == 0)}, non-OK builds {int((status != 0).sum())})", flush=True)
pb = native.ProblemBatch(specs)
ts = []
for rep in range(5):
    t0 = time.perf_counter()
    ctx.plan_problems(pb)
    ts.append(time.perf_counter() - t0)
t = min(ts)
print(f"gmt_plan_problems (ProblemBatch, flattened once): {1e3 * t:.1f} ms -> {q / t:.0f} plans/s", flush=True)
t0 = time.perf_counter()
insts = [ctx.build_instance(s) for s in specs]
b = ctx.batch(insts, 1.0)
b.launch()
s2 = b.summaries()
t1 = time.perf_counter()
print(f"per-problem builds + batched solve: {1e3 * (t1 - t0):.1f} ms -> {q / (t1 - t0):.0f} plans/s", flush=True)
same = all((a.status, a.cost, a.iterations) == (c.status, c.cost, c.iterations) for a, c in zip(summ, s2))
print("identical summaries:", same)
