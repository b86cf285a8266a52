"""configs[4] device-resident solve: shape sweep (CTAs per query x threads)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1705_02403_b200 import problem as P
from paper_1705_02403_b200.native import Context, ProblemBatch, OPT_BATCH_CLUSTER, OPT_BATCH_THREADS
Q = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
shapes = [(2, 512), (1, 512), (1, 256), (2, 256), (4, 512)]
ctx = Context(0)
pb = ProblemBatch([P.random_di_query(20171005, q, n=4000, radius=1.6) for q in range(Q)])
stream = torch.cuda.ExternalStream(ctx.stream)
ref = None
for cs, th in shapes:
    ctx.set_option(OPT_BATCH_CLUSTER, cs)
    ctx.set_option(OPT_BATCH_THREADS, th)
    b, st = ctx.batch_problems(pb)
    b.launch(); b.launch(); ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(3):
        b.launch()
    e1.record(stream); e1.synchronize()
    ms = e0.elapsed_time(e1) / 3
    s = [(x.status, x.cost, x.iterations) for x in b.summaries()]
    ref = ref or s
    print(f"cluster={cs} threads={th}: {ms:.2f} ms  {Q / ms * 1e3:.0f} plans/s  same={s == ref}", flush=True)
    b.close()
