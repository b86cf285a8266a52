"""Multi-threaded small-query throughput: N host threads, each with its own
context / stream, loop (a) plan on a prebuilt n=500 instance, (b) build +
plan + destroy.  Shows whether concurrent contexts overlap on the GPU."""
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from helpers import scene  # noqa: E402
from paper_1705_02403_b200 import native  # noqa: E402

spec = scene("rectangles_2d", 500)


def run(nthreads, mode, reps=200):
    ctxs = [native.Context(0) for _ in range(nthreads)]
    insts = [c.build_instance(spec) for c in ctxs]
    def work(i):
        c, inst = ctxs[i], insts[i]
        for _ in range(reps):
            if mode == "plan":
                c.plan(inst)
            else:
                j = c.build_instance(spec)
                c.plan(j)
                j.close() if hasattr(j, "close") else None
    ths = [threading.Thread(target=work, args=(i,)) for i in range(nthreads)]
    t0 = time.perf_counter()
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    dt = time.perf_counter() - t0
    print(f"{mode:6s} threads={nthreads:2d}: {nthreads * reps / dt:8.0f} ops/s ({dt / reps * 1e3:.2f} ms per op per thread)",
          flush=True)


for mode in ("plan", "build"):
    for n in (1, 4, 16):
        run(n, mode)
