"""Per-phase clock split of the batched C2 solve (debug build with
-DGMT_PHASE_TIMING: python tools/build_variant.py phase -DGMT_PHASE_TIMING=1,
then GMT_B200_LIB=build/variants/libgmt_b200_phase.so python tools/phase_timing.py)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_02403_b200 import native, problem as P  # noqa: E402

ctx = native.Context(0)
insts = [ctx.build_instance(P.random_forest_query(20171005, q, n=4000)) for q in range(512)]
b = ctx.batch(insts, 1.0)
b.launch()
ctx.synchronize()
ctx.set_option(native.OPT_COUNTERS, 1)
out = (C.c_int64 * 16)()
native.lib().gmt_ctx_counters(ctx.h, out, 1)
b2 = ctx.batch(insts, 1.0)
b2.launch()
native.lib().gmt_ctx_counters(ctx.h, out, 1)
ph = list(out)[4:8]
tot = sum(ph)
for name, v in zip(("P0-P3 sweeps + close", "P4 marks + barrier", "candidate list", "P5 scan/check/commit + barrier"), ph):
    print(f"{name:32s} {100 * v / tot:5.1f} %  ({v / 512 / 1965:.1f} us per query at 1965 MHz)")
