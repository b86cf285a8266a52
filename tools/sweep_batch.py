"""Timing sweep of the batched solve: batch size vs time (device-resident)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1705_02403_b200 import problem as P  # noqa: E402
from paper_1705_02403_b200.native import (Context, OPT_BATCH_CLUSTER,  # noqa: E402
                                          OPT_BATCH_THREADS)

ctx = Context(0)
stream = torch.cuda.ExternalStream(ctx.stream)
qmax = int(sys.argv[1]) if len(sys.argv) > 1 else 512
mk = P.random_di_query if os.environ.get("DI") else P.random_forest_query
insts = [ctx.build_instance(mk(20171005, q, n=4000)) for q in range(qmax)]


def timeit(b, reps=10):
    for _ in range(3):
        b.launch()
    ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        b.launch()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


for cs, thr in ((1, 256), (1, 512), (1, 384), (2, 512), (2, 256)):
    ctx.set_option(OPT_BATCH_CLUSTER, cs)
    ctx.set_option(OPT_BATCH_THREADS, thr)
    for q in (1, 148, 296, 512):
        if q > qmax:
            continue
        try:
            b = ctx.batch(insts[:q], 1.0)
            ms = timeit(b)
            print(f"cs={cs} thr={thr} q={q}: {ms:.3f} ms  {q / ms * 1e3:.0f} plans/s", flush=True)
            b.close()
        except Exception as e:
            print(f"cs={cs} thr={thr} q={q}: {e}")
