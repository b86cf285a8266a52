"""Per-phase clock split of the configs[4] batched DI solve (debug build:
python tools/build_variant.py phase -DGMT_PHASE_TIMING=1, then
GMT_B200_LIB=build/variants/libgmt_b200_phase.so python tools/di_phase.py)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_02403_b200 import native, problem as P  # noqa: E402

Q = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
ctx = native.Context(0)
pb = native.ProblemBatch([P.random_di_query(20171005, q, n=4000, radius=1.6) for q in range(Q)])
ctx.set_option(native.OPT_COUNTERS, 1)  # (results carry the counters from the batch's creation on)
b, _ = ctx.batch_problems(pb)
b.launch()
b.summaries()
ctx.synchronize()
out = (C.c_int64 * 16)()
native.lib().gmt_ctx_counters(ctx.h, out, 1)
b.launch()
native.lib().gmt_ctx_counters(ctx.h, out, 1)
ph = list(out)[4:8]
tot = sum(ph)
for name, v in zip(("P0-P3 sweeps + close", "P4 marks + barrier", "candidate list", "P5 scan/check/commit + barrier"), ph):
    print(f"thread 0: {name:32s} {100 * v / tot:5.1f} %  ({v / Q / 1965:.1f} us per query at 1965 MHz)")
w = list(out)[8:12]
nw = 24
print(f"per warp (share of thread 0's pass time): P5 loop {100 * w[0] / nw / tot:.1f} %, inside checks (group 0) "
      f"{100 * w[1] / nw / tot:.1f} %, wait at the P5 barrier {100 * w[2] / nw / tot:.1f} %, P4 loop {100 * w[3] / nw / tot:.1f} %")
