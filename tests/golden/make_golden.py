"""Generate the committed golden fixtures under tests/golden/ from the
UNMODIFIED reference (oracle/_ref/libgmtref.so, built from /root/reference)
and the reference scene files.  Run in the build container (needs
/root/reference); the outputs travel to the GPU box, the reference does not.

    python tests/golden/make_golden.py

Writes:
  scenes.json   the reference's bundled problem scenes, parsed by the
                reference's own parse_problem (problem.cpp:102-223) into flat
                fields (Euclidean scenes; forest_dubins keeps only its header)
  plans.json    known-answer GMT*/FMT* results of the reference on those
                scenes and the synthetic BASELINE scenes: status, cost bits,
                iterations, checks, path, per-pass stats, and SHA-256 digests
                of the full tree arrays and of the sample/graph arrays
  kats.json     Halton / nth_prime / radius known answers from the
                reference's tests (test_sampling.cpp:29-66, test_graph.cpp:44-89)
"""
from __future__ import annotations

import glob
import hashlib
import json
import os
import struct
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1705_02403_b200 import problem as P  # noqa: E402
from paper_1705_02403_b200.graph import Graph  # noqa: E402

SCENE_DIR = "/root/reference/proj/scenes"


def f64hex(x: float) -> str:
    return struct.pack("<d", x).hex()


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def scenes(ref):
    out = {}
    for path in sorted(glob.glob(os.path.join(SCENE_DIR, "*.json"))):
        name = os.path.basename(path)[:-5]
        text = open(path).read()
        doc = json.loads(text)
        if doc.get("schema") != "gmt-problem/1":
            continue
        if doc["steering"]["model"] != "euclidean":
            out[name] = {"steering": doc["steering"]["model"], "skipped": True}
            continue
        f = ref.parse_problem(text)
        out[name] = {
            "dim": f["dim"], "box_lo": f["box_lo"].tolist(), "box_hi": f["box_hi"].tolist(),
            "goal_lo": f["goal_lo"].tolist(), "goal_hi": f["goal_hi"].tolist(),
            "init": f["init"].tolist(), "n": f["n"], "lambda": f["lam"], "eta": f["eta"],
            "radius_override": f["radius_override"], "sampling_kind": f["sampling_kind"],
            "start_index": f["start_index"], "seed": f["seed"], "problem_key": str(f["key"]),
        }
    return out


def spec_from(entry) -> P.ProblemSpec:
    return P.ProblemSpec(dim=entry["dim"], box_lo=np.array(entry["box_lo"]).reshape(-1, entry["dim"]),
                         box_hi=np.array(entry["box_hi"]).reshape(-1, entry["dim"]),
                         goal_lo=np.array(entry["goal_lo"]), goal_hi=np.array(entry["goal_hi"]),
                         init=np.array(entry["init"]), n=entry["n"], lam=entry["lambda"],
                         eta=entry["eta"], radius_override=entry["radius_override"],
                         sampling_kind=entry["sampling_kind"], start_index=entry["start_index"],
                         seed=entry["seed"])


def plan_record(res):
    return {
        "status": int(res.status), "cost": f64hex(res.cost), "iterations": int(res.iterations),
        "checks": int(res.total_collision_checks), "path": res.path_indices.tolist(),
        "group_sizes": res.group_sizes.tolist(), "nodes_added": res.nodes_added.tolist(),
        "collision_checks": res.collision_checks.tolist(),
        "label_sha": digest(res.label), "cost_sha": digest(res.tree_cost),
        "parent_sha": digest(res.parent), "iter_added_sha": digest(res.iteration_added),
    }


def cases(sc):
    """(case name, spec) pairs: bundled scenes at BASELINE sizes + C2 forest."""
    yield "rectangles_2d_n2000", spec_from(sc["rectangles_2d"]).with_n(2000)
    yield "rectangles_2d_n250_uniform", _uniform(spec_from(sc["rectangles_2d"]).with_n(250), 42)
    yield "rectangles_3d_n1000", spec_from(sc["rectangles_3d"])
    yield "maze_3d_n1500", spec_from(sc["maze_3d"]).with_n(1500)
    yield "rectangles_6d_n600", spec_from(sc["rectangles_6d"]).with_n(600)
    yield "cave_sim", spec_from(sc["cave_sim"])
    yield "forest3d_n1000", P.forest_3d(3, 1000)


def _uniform(spec, seed):
    spec.sampling_kind = 1
    spec.seed = seed
    return spec


def main():
    ref = oracle.ref()
    sc = scenes(ref)
    json.dump(sc, open(os.path.join(HERE, "scenes.json"), "w"), indent=1)

    plans = {}
    for name, spec in cases(sc):
        inst = ref.instance_build(spec)
        info = inst.info()
        coords, gidx, ptr, col, cost = inst.download(spec.dim)
        rec = {"n": info["n"], "init_index": info["init_index"], "radius": f64hex(info["radius"]),
               "num_edges": info["num_edges"], "goal_idx": gidx.tolist(),
               "coords_sha": digest(coords), "row_ptr_sha": digest(ptr), "col_sha": digest(col),
               "cost_sha": digest(cost), "plans": {}}
        for lam in (1.0, 0.5, 0.2):
            rec["plans"][f"gmt_{lam}"] = plan_record(inst.plan(lam))
        g = Graph(info["n"], info["radius"], ptr, col, cost, dim=spec.dim)
        rec["plans"]["fmt"] = plan_record(ref.fmt_plan(spec, coords, len(gidx), g, info["init_index"]))
        plans[name] = rec
        print(name, info, rec["plans"]["gmt_1.0"]["iterations"], flush=True)
    json.dump(plans, open(os.path.join(HERE, "plans.json"), "w"), indent=1)

    kats = {
        "halton": [[i, b, f64hex(ref.halton(i, b))] for i in (1, 2, 3, 4, 5, 17, 1000, 123457)
                   for b in (2, 3, 5, 7, 29, 37)],
        "nth_prime": [[k, ref.nth_prime(k)] for k in (1, 2, 3, 4, 10, 13)],
        "radius": [[d, n, eta, mu, f64hex(ref.connection_radius(d, n, eta, mu))]
                   for d in (2, 3, 5, 6, 8, 12) for n in (100, 1000, 2000, 4000, 5000, 8000)
                   for eta, mu in ((0.0, 1.0), (0.3, 0.8))],
        "unit_ball": [[d, f64hex(ref.unit_ball_volume(d))] for d in range(1, 13)],
    }
    json.dump(kats, open(os.path.join(HERE, "kats.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
