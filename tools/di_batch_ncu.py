"""configs[4] for ncu: one launch of the device-resident 4096-query batch
(materialised rows) after its results were read once (largest-first order),
then one gmt_plan_problems call (pool views)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_02403_b200 import problem as P  # noqa: E402
from paper_1705_02403_b200.native import Context, ProblemBatch  # noqa: E402

ctx = Context(0)
pb = ProblemBatch([P.random_di_query(20171005, q, n=4000, radius=1.6) for q in range(4096)])
b, _ = ctx.batch_problems(pb)
b.launch()
b.summaries()
b.launch()
ctx.synchronize()
st, summ, _ = ctx.plan_problems(pb)
print("ok", sum(1 for s in summ if s.status == 0))
