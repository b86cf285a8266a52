"""Profiling driver: build Q forest queries on the GPU and launch the
batched solve (or one clustered single-query solve) a few times.
    python tools/profile_batch.py [--queries 512] [--single] [--launches 3]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_02403_b200 import problem as P  # noqa: E402
from paper_1705_02403_b200.native import Context, OPT_BATCH_CLUSTER  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--queries", type=int, default=512)
ap.add_argument("--n", type=int, default=4000)
ap.add_argument("--single", action="store_true")
ap.add_argument("--cluster", type=int, default=16)
ap.add_argument("--launches", type=int, default=3)
a = ap.parse_args()
ctx = Context(0)
if a.single:
    insts = [ctx.build_instance(P.forest_3d(3, a.n))]
    ctx.set_option(OPT_BATCH_CLUSTER, a.cluster)
else:
    insts = [ctx.build_instance(P.random_forest_query(20171005, q, n=a.n)) for q in range(a.queries)]
b = ctx.batch(insts, 1.0)
for _ in range(a.launches):
    b.launch()
ctx.synchronize()
s = b.summaries()
print("solved", sum(1 for x in s if x.status == 0), "/", len(s))
