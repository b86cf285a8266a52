"""configs[1] for ncu: the 512-query 3D forest batch (device-resident solve)
and one gmt_plan_problems call (batched sampling + r-disk grid + solve)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_02403_b200 import problem as P  # noqa: E402
from paper_1705_02403_b200.native import Context, ProblemBatch  # noqa: E402

ctx = Context(0)
specs = [P.random_forest_query(20171005, q, n=4000) for q in range(512)]
insts = [ctx.build_instance(s) for s in specs]
b = ctx.batch(insts, 1.0)
b.launch()
ctx.synchronize()
st, summ, _ = ctx.plan_problems(ProblemBatch(specs))
print("ok", sum(1 for s in summ if s.status == 0))
