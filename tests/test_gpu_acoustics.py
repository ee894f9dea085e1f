"""Full-size multi-step property ("its amplitude will drop off
inversely proportional to the distance traveled"): the C3 pulse stepped to the outer boundary
(1,318 LSERK4 steps at CFL 0.5 on 662k elements, the bench's launch configuration) must decay
like 1/r along a free ray -- a property of the exact solution that holds at any size, checked on
the stepped GPU solution where the oracle cannot follow; and the pass-through boundary must not
raise the near-boundary spectrum above spherical spreading (no reflection, reading A6)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))


@pytest.mark.gpu
def test_c3_pulse_decays_like_one_over_r():
    import reflection_study as rs
    r = rs.run("C3")
    assert all(e >= 0 for e in r["sensor_elements"])
    assert abs(r["decay"]["exponent"] + 1.0) < 0.05, r["decay"]
    refl = r["reflection"]
    assert refl["mean_db_difference"] < refl["spreading_only_db"] + 1.0, refl
