"""configs[1] 512-query forest batch: solve time per batch shape (CTAs per
query x threads), device-resident, largest-first order after a summaries()
read, as bench.py does.  python tools/forest_sweep.py [CSxTHREADS ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1705_02403_b200 import problem as P  # noqa: E402
from paper_1705_02403_b200.native import OPT_BATCH_CLUSTER, OPT_BATCH_THREADS, Context  # noqa: E402

ctx = Context(0)
stream = torch.cuda.ExternalStream(ctx.stream)
specs = [P.random_forest_query(20171005, q, n=4000) for q in range(512)]
insts = [ctx.build_instance(s) for s in specs]
shapes = [tuple(map(int, a.split("x"))) for a in sys.argv[1:]] or [(0, 0), (1, 512), (2, 256), (2, 512), (4, 512)]
ref = None
for cs, th in shapes:
    ctx.set_option(OPT_BATCH_CLUSTER, cs)
    ctx.set_option(OPT_BATCH_THREADS, th)
    b = ctx.batch(insts, 1.0)
    b.launch()
    s = [(x.status, x.cost, x.iterations) for x in b.summaries()]
    b.launch()
    ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(5):
        b.launch()
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 5
    ref = ref or s
    print(f"cluster={cs} threads={th}: {ms:.3f} ms  {len(specs) / ms * 1e3:.0f} plans/s  same={s == ref}", flush=True)
    b.close()
