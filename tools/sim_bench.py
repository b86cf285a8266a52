"""Replanning-simulator campaign throughput (simulator.cpp:178-227): the
device path (every replan on the B200, host worker threads each with a
stream) against the reference's CPU campaign on all host cores.
    python tools/sim_bench.py [trials_per_cell] [workers]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import oracle  # noqa: E402  (the reference arm only)
from helpers import scene  # noqa: E402
from paper_1705_02403_b200 import native, problem as P  # noqa: E402

trials = int(sys.argv[1]) if len(sys.argv) > 1 else 10
workers = int(sys.argv[2]) if len(sys.argv) > 2 else (os.cpu_count() or 8)
n = int(sys.argv[3]) if len(sys.argv) > 3 else 500
sc = P.Scenario(scene("rectangles_2d", n), robot_speed=0.2, time_limit=12.0, trials=trials, seed=3)
lat, rates, sig = [0.1, 0.2, 0.4], [0.0, 2.0, 5.0], [0.0, 0.02]
t0 = time.perf_counter()
got = native.run_campaign(sc, lat, rates, sig, workers=workers)
t1 = time.perf_counter()
want = oracle.ref().run_campaign(sc, lat, rates, sig, workers=os.cpu_count() or 8)
t2 = time.perf_counter()
print(f"n={n} cells={got.size} trials/cell={trials} workers={workers} identical={np.array_equal(got, want)}")
print(f"device campaign {t1 - t0:.2f} s, reference CPU campaign ({os.cpu_count()} threads) {t2 - t1:.2f} s, "
      f"speed-up {(t2 - t1) / (t1 - t0):.2f}x; successes {int(got.sum())}/{got.size * trials}")
