"""The C-ABI scene loader (gmt_problem_parse / gmt_problem_load,
csrc/problem_file.cpp) against the reference's own parse_problem
(problem.cpp:102-231, compiled into oracle/_ref): every bundled scene
(tests/golden/scene_texts.json, the reference's proj/scenes) parses to the
same fields bit for bit, and every malformed variant fails with the same
path-named InvalidInputError message.  The Python loader (problem.py) is held
to the same bar.  CPU only: parsing needs no device."""
import json
import os

import numpy as np
import pytest

from paper_1705_02403_b200 import abi, native, problem as P
from paper_1705_02403_b200.errors import InvalidInputError
from helpers import GOLDEN

with open(os.path.join(GOLDEN, "scene_texts.json")) as f:
    SCENES = json.load(f)


def _ref_error(ref, text):
    try:
        ref.parse_problem(text)
    except InvalidInputError as e:
        return str(e)
    return None


def _error(fn, text):
    try:
        fn(text)
    except InvalidInputError as e:
        return str(e)
    return None


def _same_fields(spec, want):
    d = want["dim"]
    assert spec.dim == d
    assert spec.box_lo.reshape(-1, d).tobytes() == want["box_lo"].tobytes()
    assert spec.box_hi.reshape(-1, d).tobytes() == want["box_hi"].tobytes()
    assert np.asarray(spec.goal_lo).tobytes() == want["goal_lo"].tobytes()
    assert np.asarray(spec.goal_hi).tobytes() == want["goal_hi"].tobytes()
    assert np.asarray(spec.init, np.float64).tobytes() == want["init"].tobytes()
    assert (spec.n, spec.lam, spec.eta, spec.radius_override) == \
        (want["n"], want["lam"], want["eta"], want["radius_override"])
    assert (spec.sampling_kind, spec.start_index, spec.seed, spec.steering) == \
        (want["sampling_kind"], want["start_index"], want["seed"], want["steering"])


@pytest.mark.parametrize("name", sorted(SCENES))
def test_bundled_scenes_match_reference(ref, name):
    text = SCENES[name]
    err = _ref_error(ref, text)
    if err is not None:  # cave_campaign.json is a campaign file, not a problem
        assert _error(native.parse_problem, text) == err
        assert _error(P.parse_problem, text) == err
        return
    want = ref.parse_problem(text)
    _same_fields(native.parse_problem(text), want)
    _same_fields(P.parse_problem(text), want)


def test_load_problem(tmp_path, ref):
    text = SCENES["maze_3d"]
    path = tmp_path / "maze_3d.json"
    path.write_text(text)
    _same_fields(native.load_problem(str(path)), ref.parse_problem(text))
    missing = str(tmp_path / "nope.json")
    with pytest.raises(InvalidInputError, match="cannot open file"):
        native.load_problem(missing)


BASE = json.loads(SCENES["rectangles_2d"])


def _variant(**edits):
    doc = json.loads(json.dumps(BASE))
    for path, value in edits.items():
        node, keys = doc, path.split("__")
        for k in keys[:-1]:
            node = node[int(k)] if isinstance(node, list) else node[k]
        last = keys[-1]
        if value is _DROP:
            if isinstance(node, list):
                node.pop(int(last))
            else:
                node.pop(last)
        elif isinstance(node, list):
            node[int(last)] = value
        else:
            node[last] = value
    return json.dumps(doc)


_DROP = object()

ERROR_CASES = {
    "unknown_top": _variant(dimensions=2),
    "missing_n": _variant(n=_DROP),
    "n_zero": _variant(n=0),
    "n_float": _variant(n=50.0),
    "n_string": _variant(n="50"),
    "lambda_zero": _variant(**{"lambda": 0.0}),
    "lambda_big": _variant(**{"lambda": 1.5}),
    "eta_negative": _variant(eta=-0.5),
    "radius_negative": _variant(radius_override=-1.0),
    "radius_zero": _variant(radius_override=0),
    "schema": _variant(schema="gmt-problem/2"),
    "schema_type": _variant(schema=1),
    "dimension_zero": _variant(dimension=0),
    "dimension_float": _variant(dimension=2.0),
    "box_order": _variant(obstacles__0__lo=[0.5, 0.5], obstacles__0__hi=[0.4, 0.9]),
    "box_short": _variant(obstacles__1__lo=[0.5]),
    "box_unknown": _variant(obstacles__0__mid=[0.5, 0.5]),
    "box_not_object": _variant(obstacles__2=[0.1, 0.2]),
    "box_bad_number": _variant(obstacles__0__hi=[0.4, "x"]),
    "obstacles_type": _variant(obstacles={"lo": [0, 0]}),
    "init_blocked": _variant(init={"coords": [0.3, 0.3]}),
    "init_outside": _variant(init={"coords": [1.2, 0.3]}),
    "init_heading": _variant(init={"coords": [0.05, 0.3], "heading": 0.0}),
    "init_unknown": _variant(init={"coords": [0.05, 0.3], "speed": 1}),
    "goal_missing_hi": _variant(goal={"lo": [0.9, 0.2]}),
    "model": _variant(steering={"model": "reeds_shepp"}),
    "rho_on_euclidean": _variant(steering={"model": "euclidean", "rho": 0.1}),
    "steering_unknown": _variant(steering={"model": "euclidean", "turn": 1}),
    "dubins_needs_heading": _variant(steering={"model": "dubins_airplane"}),
    "sampling_seed_on_halton": _variant(sampling={"kind": "halton", "seed": 3}),
    "sampling_start_zero": _variant(sampling={"kind": "halton", "start_index": 0}),
    "sampling_start_on_uniform": _variant(sampling={"kind": "uniform", "start_index": 4}),
    "sampling_kind": _variant(sampling={"kind": "sobol"}),
    "sampling_negative_seed": _variant(sampling={"kind": "uniform", "seed": -1}),
    "notes_type": _variant(notes=3),
    "top_array": "[1, 2]",
    "empty": "",
    "trailing_comma": '{"schema": "gmt-problem/1",}',
    "truncated": SCENES["rectangles_2d"][:40],
    "garbage_after": SCENES["rectangles_2d"] + " x",
}


@pytest.mark.parametrize("case", sorted(ERROR_CASES))
def test_errors_match_reference(ref, case):
    text = ERROR_CASES[case]
    want = _ref_error(ref, text)
    assert want is not None, f"the reference accepts {case}"
    got = _error(native.parse_problem, text)
    py = _error(P.parse_problem, text)
    if want.startswith("invalid JSON"):   # the JSON readers' own wording differs
        assert got is not None and got.startswith("invalid JSON")
        assert py is not None and py.startswith("invalid JSON")
    else:
        assert got == want
        assert py == want


def test_accepted_variants_match_reference(ref):
    """Forms the reference accepts: integers where doubles are expected,
    exponents, a repeated key (the last value wins), unicode notes, uniform
    sampling with a large seed, dubins with its optional fields."""
    texts = [
        _variant(**{"lambda": 1}, eta=0, radius_override=2),
        _variant(radius_override=1.5e-1, sampling={"kind": "halton", "start_index": 18446744073709551615}),
        _variant(sampling={"kind": "uniform", "seed": 18446744073709551615}),
        SCENES["rectangles_2d"].replace('"n"', '"n": 7, "n"', 1),
        _variant(notes="pillars é中 \\ \"q\""),
        _variant(steering={"model": "dubins_airplane", "rho": 0.2, "discretization_step": 0,
                           "planar_cost_only": True},
                 init={"coords": [0.05, 0.3], "heading": 1}),
    ]
    for t in texts:
        want = ref.parse_problem(t)
        _same_fields(native.parse_problem(t), want)
        _same_fields(P.parse_problem(t), want)
