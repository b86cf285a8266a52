"""Small solves through every solve-kernel shape (single CTA narrow / wide,
2/8/16-CTA clusters; Euclidean D = 3, double integrator D = 6), the batched
offline builders (r-disk grid pass) and the shared-pool derivation, each
repeated --repeats times (tests/test_gpu_sanitizer.py).  Exit 0 when every
result matches the single-CTA baseline bit for bit; prints a digest of the
batched summaries (identical across runs unless something races)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_02403_b200 import abi, problem as P  # noqa: E402
from paper_1705_02403_b200.native import (OPT_BATCH_CLUSTER, OPT_BATCH_THREADS, OPT_CLUSTER,  # noqa: E402
                                          Context)

import argparse
import hashlib

ap = argparse.ArgumentParser()
ap.add_argument("--repeats", type=int, default=1)
args = ap.parse_args()
ctx = Context(0)
bad = 0
for _ in range(args.repeats):
    for spec in (P.forest_3d(3, 500), P.di_forest(3, 300, radius=2.6)):
        inst = ctx.build_instance(spec)
        base = None
        for cs in (1, 2, 8, 16):
            ctx.set_option(OPT_CLUSTER, cs)
            r = ctx.plan(inst)
            base = base or r
            if abi.full_parity(r, base):
                bad += 1
                print("cluster", cs, "differs", abi.full_parity(r, base))
        ctx.set_option(OPT_CLUSTER, 0)
        for th in (256, 512):  # batched single-CTA shapes (narrow / wide)
            ctx.set_option(OPT_BATCH_CLUSTER, 1)
            ctx.set_option(OPT_BATCH_THREADS, th)
            b = ctx.batch([inst, inst], 1.0)
            b.launch()
            if abi.full_parity(b.result(1), base):
                bad += 1
                print("batch", th, "differs")
            b.close()
        ctx.set_option(OPT_BATCH_CLUSTER, 0)
        ctx.set_option(OPT_BATCH_THREADS, 0)
digests = set()
for _ in range(args.repeats):
    h = hashlib.sha256()
    st, summ, _ = ctx.plan_problems([P.random_forest_query(7, q, n=400) for q in range(16)])
    st2, summ2, _ = ctx.plan_problems([P.random_di_query(7, q, n=300, radius=2.6) for q in range(16)])
    for s in list(summ) + list(summ2):
        h.update(repr((s.status, s.cost, s.iterations, s.total_collision_checks, s.path_len)).encode())
    digests.add(h.hexdigest())
if len(digests) != 1:
    bad += 1
print("batched digest", sorted(digests))
print("mismatches", bad)
sys.exit(1 if bad else 0)
