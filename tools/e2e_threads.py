"""gmt_plan_problems from S host threads (one context each) vs one thread."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_02403_b200 import native, problem as P  # noqa: E402

Q, CALLS = 512, 16
pb = native.ProblemBatch([P.random_forest_query(20171005, i, n=4000) for i in range(Q)])
ctxs = [native.Context(0) for _ in range(3)]
for c in ctxs:
    for _ in range(2):
        c.plan_problems(pb)
for S in (1, 2, 3):
    def work(c, k):
        for _ in range(k):
            c.plan_problems(pb)
    th = [threading.Thread(target=work, args=(ctxs[i], CALLS // S)) for i in range(S)]
    t0 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    dt = time.perf_counter() - t0
    n = (CALLS // S) * S
    print(f"threads {S}: {1e3 * dt / n:.2f} ms per call -> {Q * n / dt:.0f} plans/s", flush=True)
