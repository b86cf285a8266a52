"""GMTG v1 graph-cache interop and problem_key (
graph.cpp:190-343, problem.cpp:281-303).  Host-side C ABI calls checked
against the unmodified reference: identical keys, byte-identical files in
both directions, and the same hit / miss verdict on every corruption the
reference's loader rejects."""
import numpy as np
import pytest

from paper_1705_02403_b200 import abi, native, problem as P
from paper_1705_02403_b200.graph import Graph
from helpers import SCENE_NAMES, forest_dubins, oracle_instance, scene


def _specs():
    out = [scene(s) for s in SCENE_NAMES]
    u = scene("rectangles_2d", 300)
    u.sampling_kind, u.seed = abi.SAMPLE_UNIFORM, 12345
    out.append(u)
    out.append(P.forest_3d(3, 700))
    h = scene("rectangles_3d", 500)
    h.start_index = 17
    out.append(h)
    return out


def test_problem_key_matches_reference(ref):
    keys = set()
    for spec in _specs():
        k = native.problem_key(spec)
        assert k == ref.problem_key(spec)
        keys.add(k)
    assert len(keys) == len(_specs())  # every field change moves the key


def test_problem_key_dubins_matches_reference(ref):
    """Dubins problems key on kind, rho, step() and planar_cost_only
    (problem.cpp:284-287) and carry with_heading (problem.cpp:197)."""
    specs = [forest_dubins()]
    for f, v in (("dubins_rho", 0.1), ("dubins_step", 0.004), ("dubins_planar", 1)):
        s = forest_dubins()
        setattr(s, f, v)
        specs.append(s)
    keys = {native.problem_key(s) for s in specs}
    assert len(keys) == len(specs)
    for s in specs:
        assert native.problem_key(s) == ref.problem_key(s)


def test_problem_key_rejects_kinodynamic():
    spec = P.di_forest(3, 200)
    with pytest.raises(Exception):
        native.problem_key(spec)


@pytest.mark.parametrize("name,n", [("rectangles_2d", 800), ("maze_3d", 900), ("rectangles_6d", 400)])
def test_cache_files_interchange_with_reference(tmp_path, port, ref, name, n):
    spec = scene(name, n)
    key = native.problem_key(spec)
    inst = oracle_instance(port, spec)
    g = inst["graph"]
    ours = tmp_path / "ours.gmtg"
    native.graph_cache_save(str(ours), key, g)
    # the reference loads our file and gets the same graph
    got = ref.load_graph_cache(str(ours), key, inst["coords"], inst["radius"])
    assert got is not None
    assert np.array_equal(got[0], g.out_ptr) and np.array_equal(got[1], g.out_col)
    assert got[2].tobytes() == g.out_cost.tobytes()
    # the reference's own file for the same problem is byte-identical
    theirs = tmp_path / "theirs.gmtg"
    ri = ref.instance_build(spec)
    assert ri.save_cache(str(theirs), key)
    assert ours.read_bytes() == theirs.read_bytes()
    # and we load the reference's file
    back = native.graph_cache_load(str(theirs), key, g.n, g.radius)
    assert back is not None and np.array_equal(back.out_col, g.out_col)
    assert back.out_cost.tobytes() == g.out_cost.tobytes()


def test_cache_miss_verdicts_match_reference(tmp_path, port, ref):
    spec = scene("rectangles_2d", 400)
    key = native.problem_key(spec)
    inst = oracle_instance(port, spec)
    g, coords, r = inst["graph"], inst["coords"], inst["radius"]
    good = tmp_path / "g.gmtg"
    native.graph_cache_save(str(good), key, g)
    data = good.read_bytes()
    header = 4 + 4 + 8 + 4 + 8 + 1 + 8 + 8 + 1
    first_row = header + 4  # first (target, cost) pair of row 0

    def variant(name, blob):
        f = tmp_path / name
        f.write_bytes(blob)
        return str(f)

    row0 = int(g.out_ptr[1] - g.out_ptr[0])
    assert row0 >= 2
    bad_order = bytearray(data)  # swap the first two targets of row 0
    t0, t1 = bytes(bad_order[first_row:first_row + 4]), bytes(bad_order[first_row + 12:first_row + 16])
    bad_order[first_row:first_row + 4], bad_order[first_row + 12:first_row + 16] = t1, t0
    cases = {
        "ok": (str(good), key, r),
        "missing": (str(tmp_path / "none.gmtg"), key, r),
        "key": (str(good), key ^ 1, r),
        "radius": (str(good), key, np.nextafter(r, 1.0)),
        "magic": (variant("m", b"XMTG" + data[4:]), key, r),
        "version": (variant("v", data[:4] + b"\x02" + data[5:]), key, r),
        "truncated": (variant("t", data[:-3]), key, r),
        "trailing": (variant("x", data + b"\x00"), key, r),
        "dubins": (variant("d", data[:header - 18] + b"\x01" + data[header - 17:]), key, r),
        "order": (variant("o", bytes(bad_order)), key, r),
    }
    for name, (f, k, rad) in cases.items():
        want = ref.load_graph_cache(f, k, coords, rad) is not None
        got = native.graph_cache_load(f, k, g.n, rad) is not None
        assert got == want, name
        assert got == (name == "ok"), name
    # a different n is a miss too
    assert native.graph_cache_load(str(good), key, g.n - 1, r) is None
    assert ref.load_graph_cache(str(good), key, coords[:-1], r) is None


def test_empty_graph_roundtrip(tmp_path):
    g = Graph(3, 0.01, np.zeros(4, np.int64), np.zeros(0, np.int32), np.zeros(0))
    f = tmp_path / "e.gmtg"
    native.graph_cache_save(str(f), 7, g)
    back = native.graph_cache_load(str(f), 7, 3, 0.01)
    assert back is not None and back.num_edges == 0
