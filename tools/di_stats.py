"""configs[4]: work counts of the batched DI solve (checks, passes, row scans)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1705_02403_b200 import problem as P
from paper_1705_02403_b200.native import Context, ProblemBatch, OPT_BATCH_CLUSTER, OPT_BATCH_THREADS, OPT_COUNTERS
Q = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
ctx = Context(0)
pb = ProblemBatch([P.random_di_query(20171005, q, n=4000, radius=1.6) for q in range(Q)])
ctx.set_option(OPT_BATCH_CLUSTER, 1)
ctx.set_option(OPT_BATCH_THREADS, 256)
ctx.set_option(OPT_COUNTERS, 1)
ctx.counters(reset=True)
b, st = ctx.batch_problems(pb)
b.launch()
cnt = ctx.counters(reset=True)
s = b.summaries()
checks = np.array([x.total_collision_checks for x in s]); it = np.array([x.iterations for x in s])
ns = np.array([x.num_stats for x in s])
print("queries", Q, "success", sum(1 for x in s if x.status == 0))
print("checks total %d mean %.0f max %d" % (checks.sum(), checks.mean(), checks.max()))
print("iterations mean %.1f max %d passes mean %.1f max %d" % (it.mean(), it.max(), ns.mean(), ns.max()))
print("counters", cnt)
