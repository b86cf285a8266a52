"""Debug helper: per-pass GPU vs oracle stats for one scene."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle
from helpers import scene, oracle_instance
from paper_1705_02403_b200.native import Context, OPT_CLUSTER

name = sys.argv[1] if len(sys.argv) > 1 else "rectangles_2d"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
cs = int(sys.argv[3]) if len(sys.argv) > 3 else 1
port = oracle.port()
spec = scene(name, n)
o = oracle_instance(port, spec)
ctx = Context(0)
ctx.set_option(OPT_CLUSTER, cs)
inst = ctx.upload(spec, o["coords"], len(o["goal_idx"]), o["graph"])
got = ctx.plan(inst, o["init"], 1.0, o["radius"])
want = port.gmt_plan(spec, o["coords"], len(o["goal_idx"]), o["graph"], o["init"], 1.0, o["radius"])
print("gpu", got, "\nref", want)
for k in range(max(len(got.group_sizes), len(want.group_sizes))):
    a = (got.group_sizes[k], got.nodes_added[k], got.collision_checks[k]) if k < len(got.group_sizes) else None
    b = (want.group_sizes[k], want.nodes_added[k], want.collision_checks[k]) if k < len(want.group_sizes) else None
    print(k, a, b, "" if a == b else "<<<")
diff = np.nonzero((got.label != want.label) | (got.parent != want.parent))[0]
print("differing nodes:", len(diff), diff[:20])
for v in diff[:10]:
    print(v, "gpu", got.label[v], got.parent[v], got.tree_cost[v], got.iteration_added[v], "| ref", want.label[v], want.parent[v], want.tree_cost[v], want.iteration_added[v])
