"""A/B timing of the batched C2 solve for one library build (select it with
GMT_B200_LIB=...): 512 forest3d n=4000 queries, median of 7 x 5 launches.
    GMT_B200_LIB=build/variants/libX.so python tools/ab_time.py [queries]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1705_02403_b200 import problem as P  # noqa: E402
from paper_1705_02403_b200.native import Context, OPT_BATCH_THREADS  # noqa: E402

q = int(sys.argv[1]) if len(sys.argv) > 1 else 512
ctx = Context(0)
if os.environ.get("BATCH_THREADS"):
    ctx.set_option(OPT_BATCH_THREADS, int(os.environ["BATCH_THREADS"]))
stream = torch.cuda.ExternalStream(ctx.stream)
insts = [ctx.build_instance(P.random_forest_query(20171005, i, n=4000)) for i in range(q)]
b = ctx.batch(insts, 1.0)
for _ in range(3):
    b.launch()
ctx.synchronize()
ts = []
for _ in range(7):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(5):
        b.launch()
    e1.record(stream)
    e1.synchronize()
    ts.append(e0.elapsed_time(e1) / 5)
s = b.summaries()
print(f"{os.environ.get('GMT_B200_LIB', 'in-tree')} thr={os.environ.get('BATCH_THREADS', 'auto')}: {statistics.median(ts):.3f} ms/launch "
      f"(min {min(ts):.3f}) solved {sum(1 for x in s if x.status == 0)}/{len(s)}", flush=True)
