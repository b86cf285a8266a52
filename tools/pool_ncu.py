"""One configs[4] plan_problems call (for ncu): Q random 6D DI queries."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_02403_b200 import problem as P
from paper_1705_02403_b200.native import Context, ProblemBatch
Q = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
ctx = Context(0)
pb = ProblemBatch([P.random_di_query(20171005, q, n=4000, radius=1.6) for q in range(Q)])
for _ in range(2):
    st, summ, _ = ctx.plan_problems(pb)
print("ok", int((st == 0).sum()), sum(1 for s in summ if s.status == 0))
