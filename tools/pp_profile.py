"""Kernel time breakdown of one gmt_plan_problems call (CUPTI via
torch.profiler; times are per kernel name, summed over the call)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1705_02403_b200 import native, problem as P  # noqa: E402

q = int(sys.argv[1]) if len(sys.argv) > 1 else 512
ctx = native.Context(0)
pb = native.ProblemBatch([P.random_forest_query(20171005, i, n=4000) for i in range(q)])
for _ in range(3):
    ctx.plan_problems(pb)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    ctx.plan_problems(pb)
    torch.cuda.synchronize()
rows = [(e.key, e.device_time_total / 1e3) for e in prof.key_averages() if e.device_time_total > 0]
for k, ms in sorted(rows, key=lambda x: -x[1]):
    print(f"{ms:9.3f} ms  {k[:100]}")
print(f"{sum(ms for _, ms in rows):9.3f} ms  total")
