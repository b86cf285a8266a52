"""One gmt_plan_problems call over 512 C2 problems (for kernel timing lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_02403_b200 import native, problem as P  # noqa: E402

ctx = native.Context(0)
specs = [P.random_forest_query(20171005, i, n=4000) for i in range(512)]
for _ in range(2):
    status, summ, _ = ctx.plan_problems(specs)
print("solved", sum(1 for s in summ if s.status == 0))
