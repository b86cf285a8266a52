"""GPU parity of the replanning simulator (simulator.cpp:66-227; SURVEY.md
§8(f) row 3): every replan (sample_free with a fresh uniform seed ->
append_init -> graph -> gmt_plan) runs on the device; the trial outcomes
and the travelled paths equal the unmodified reference's bit for bit, and a
campaign grid's success counts match."""
import numpy as np
import pytest

from paper_1705_02403_b200 import abi, native, problem as P
from helpers import scene

pytestmark = pytest.mark.gpu


def _scenario(**kw):
    return P.Scenario(scene("rectangles_2d", 300), robot_speed=0.2, time_limit=12.0, **kw)


@pytest.mark.parametrize("rate,sigma,latency", [(0.0, 0.0, 0.1), (2.0, 0.01, 0.1), (5.0, 0.02, 0.25),
                                                (1.0, 0.05, 0.05)])
def test_trials_match_reference(ctx, ref, rate, sigma, latency):
    sc = _scenario(collapse_rate=rate, disturbance_sigma=sigma, replan_latency=latency)
    results = set()
    for seed in (11, 12, 13, 14):
        a, pa = ctx.run_trial(sc, seed)
        b, pb = ref.run_trial(sc, seed)
        for f in ("result", "replans", "spawned", "noise_outliers", "time", "path_len"):
            assert getattr(a, f) == getattr(b, f), (f, seed)
        assert pa.tobytes() == pb.tobytes()
        results.add(a.result)
    if rate > 0:
        assert results & {abi.TRIAL_REACHED_GOAL, abi.TRIAL_COLLIDED}


def test_campaign_matches_reference(ref):
    sc = _scenario(trials=3, seed=7)
    lat, rates, sig = [0.1, 0.3], [0.0, 3.0], [0.0, 0.02]
    want = ref.run_campaign(sc, lat, rates, sig, workers=8)
    got = native.run_campaign(sc, lat, rates, sig, workers=6)
    assert np.array_equal(got, want)
    assert want.sum() > 0
