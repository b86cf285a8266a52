"""CPU: the gmt-problem/1 loader accepts dubins_airplane problems with the
reference's field rules (problem.cpp:132-173)."""
import pytest

from paper_1705_02403_b200 import abi, problem as P
from paper_1705_02403_b200.errors import InvalidInputError


def test_dubins_problem_json_roundtrip():
    text = """{"schema": "gmt-problem/1", "dimension": 3,
      "steering": {"model": "dubins_airplane", "rho": 0.1, "discretization_step": 0.02},
      "obstacles": [], "init": {"coords": [0.1, 0.1, 0.5], "heading": 1.0},
      "goal": {"lo": [0.8, 0.8, 0.4], "hi": [0.9, 0.9, 0.6]}, "n": 50}"""
    spec = P.parse_problem(text)
    assert spec.steering == abi.STEER_DUBINS_AIRPLANE and spec.init_heading == 1.0
    assert spec.dubins_rho == 0.1 and spec.dubins_step == 0.02


def test_dubins_problem_field_rules():
    base = """{"schema": "gmt-problem/1", "dimension": %d,
      "steering": {"model": "dubins_airplane"%s}, "obstacles": [],
      "init": {"coords": %s%s}, "goal": {"lo": [0.8, 0.8], "hi": [0.9, 0.9]}, "n": 50}"""
    with pytest.raises(InvalidInputError):   # heading required
        P.parse_problem(base % (2, "", "[0.1, 0.1]", ""))
    with pytest.raises(InvalidInputError):   # rho must be positive
        P.parse_problem(base % (2, ', "rho": 0', "[0.1, 0.1]", ', "heading": 0'))
    with pytest.raises(InvalidInputError):   # planar_cost_only must be a boolean
        P.parse_problem(base % (2, ', "planar_cost_only": 1', "[0.1, 0.1]", ', "heading": 0'))
    s = P.parse_problem(base % (2, "", "[0.1, 0.1]", ', "heading": 0.5'))
    assert s.dubins_rho == 0.1 and s.source().with_heading == 1
