"""Does the batched solve leave the GPU idle behind its slowest query?
K launches of the 512-query batch on one stream vs alternated over S
contexts (streams), wall time with a sync on both sides."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_02403_b200 import problem as P  # noqa: E402
from paper_1705_02403_b200.native import Context  # noqa: E402

K = 40
ctxs = [Context(0) for _ in range(4)]
if os.environ.get("BATCH_THREADS"):
    from paper_1705_02403_b200.native import OPT_BATCH_THREADS
    for c in ctxs:
        c.set_option(OPT_BATCH_THREADS, int(os.environ["BATCH_THREADS"]))
insts = [ctxs[0].build_instance(P.random_forest_query(20171005, q, n=4000)) for q in range(512)]
ctxs[0].synchronize()
for S in (1, 2, 3, 4):
    bs = [ctxs[i].batch(insts, 1.0) for i in range(S)]
    for b in bs:
        b.launch()
    for c in ctxs:
        c.synchronize()
    t0 = time.perf_counter()
    for k in range(K):
        bs[k % S].launch()
    for c in ctxs:
        c.synchronize()
    dt = time.perf_counter() - t0
    print(f"streams {S}: {1e3 * dt / K:.3f} ms per 512-query launch -> {512 * K / dt:.0f} plans/s", flush=True)
    for b in bs:
        b.close()
