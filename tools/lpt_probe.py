"""Does launch order matter for the 4096-query DI batch (one-wave tail)?
Queries in index order vs sorted by their collision checks (largest first)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1705_02403_b200 import problem as P
from paper_1705_02403_b200.native import Context, ProblemBatch
ctx = Context(0)
stream = torch.cuda.ExternalStream(ctx.stream)
specs = [P.random_di_query(20171005, q, n=4000, radius=1.6) for q in range(4096)]

def timed(b):
    b.launch(); ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(5):
        b.launch()
    e1.record(stream); e1.synchronize()
    return e0.elapsed_time(e1) / 5

b, _ = ctx.batch_problems(specs)
t0 = timed(b)
s = b.summaries()
work = [x.total_collision_checks for x in s]
b.close()
order = sorted(range(len(specs)), key=lambda q: -work[q])
b2, _ = ctx.batch_problems([specs[q] for q in order])
t1 = timed(b2)
b2.close()
import random
random.seed(1)
rnd = list(range(len(specs))); random.shuffle(rnd)
b3, _ = ctx.batch_problems([specs[q] for q in rnd])
t2 = timed(b3)
print(f"index order {t0:.2f} ms, largest-first {t1:.2f} ms, random {t2:.2f} ms; checks max {max(work)} mean {sum(work)/len(work):.0f}")
