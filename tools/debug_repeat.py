import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle
from helpers import scene, oracle_instance
from paper_1705_02403_b200 import abi
from paper_1705_02403_b200.native import Context, OPT_CLUSTER
port = oracle.port()
ctx = Context(0)
for name, n in [("rectangles_2d", 2000), ("maze_3d", 2000)]:
    spec = scene(name, n)
    o = oracle_instance(port, spec)
    inst = ctx.upload(spec, o["coords"], len(o["goal_idx"]), o["graph"])
    want = port.gmt_plan(spec, o["coords"], len(o["goal_idx"]), o["graph"], o["init"], 1.0, o["radius"])
    for cs in (1, 2, 4, 8, 16):
        ctx.set_option(OPT_CLUSTER, cs)
        res = []
        for rep in range(20):
            got = ctx.plan(inst, o["init"], 1.0, o["radius"])
            bad = abi.full_parity(got, want)
            res.append((got.total_collision_checks, tuple(bad)))
        print(name, cs, "ok" if all(not b for _, b in res) else res)
