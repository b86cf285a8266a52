"""configs[3] for ncu: the 12D quadrotor single solve (n = 8000) as the bench
times it (one 16-CTA cluster batch launch), after a warm-up launch.  Prints
the plan's per-pass stats."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_02403_b200 import problem as P  # noqa: E402
from paper_1705_02403_b200.native import OPT_BATCH_CLUSTER, OPT_BATCH_THREADS, Context  # noqa: E402

ctx = Context(0)
inst = ctx.build_instance(P.quad_scene())
r = ctx.plan(inst)
print("status", r.status, "iters", r.iterations, "checks", r.total_collision_checks, "n", inst.n,
      "edges", inst.num_edges)
print("groups", list(r.group_sizes), "\nadded", list(r.nodes_added), "\nchecks", list(r.collision_checks))
cs = int(os.environ.get("CS", "16"))
ctx.set_option(OPT_BATCH_CLUSTER, cs)
ctx.set_option(OPT_BATCH_THREADS, int(os.environ.get("THREADS", "0")))
b = ctx.batch([inst], 1.0)
b.launch()
ctx.synchronize()
b.launch()
ctx.synchronize()
print("ok")
