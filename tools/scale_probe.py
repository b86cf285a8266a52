"""Strong-scaling proxy on one GPU: the per-GPU share of the 4096-query
configs[4] step at N = 1, 2, 4, 8 (4096 / N queries), device-resident, with
the batch's adaptive largest-first order (results read once)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1705_02403_b200 import problem as P
from paper_1705_02403_b200.native import Context, OPT_BATCH_CLUSTER, OPT_BATCH_THREADS
from paper_1705_02403_b200.shard import shard_range
ctx = Context(0)
stream = torch.cuda.ExternalStream(ctx.stream)
base = None
shapes = [(0, 0)] + [tuple(map(int, a.split("x"))) for a in sys.argv[1:]]
for N in (1, 2, 4, 8):
    for cs, th in shapes:
        ctx.set_option(OPT_BATCH_CLUSTER, cs)
        ctx.set_option(OPT_BATCH_THREADS, th)
        specs = [P.random_di_query(20171005, q, n=4000, radius=1.6) for q in shard_range(4096, N, N - 1)]
        b, _ = ctx.batch_problems(specs)
        b.launch(); b.summaries(); b.launch(); ctx.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(10):
            b.launch()
        e1.record(stream); e1.synchronize()
        ms = e0.elapsed_time(e1) / 10
        if N == 1 and cs == 0:
            base = ms
        print(f"N={N} ({len(specs)} queries/GPU) shape={cs}x{th}: {ms:.2f} ms -> speedup {base / ms:.2f}x", flush=True)
        b.close()
