"""Host-side checks of bench.py's work model and roofline selection:
the algorithmic flops / bytes per element per stage, and which roofline binds at each order."""
import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def test_work_model_matches_design():
    # C4 (N = 4): 69,675 flop and 5,824 B per element per stage; C5 (N = 6): 330,540 / 13,664;
    # N = 1 (the paper's order): 2,940 / 864
    assert bench.flops_per_elem_stage(4) == 69675 and bench.bytes_per_elem_stage(4) == 5824
    assert bench.flops_per_elem_stage(6) == 330540 and bench.bytes_per_elem_stage(6) == 13664
    assert bench.flops_per_elem_stage(1) == 2940 and bench.bytes_per_elem_stage(1) == 864
    assert bench.flops_per_elem_stage_modal(1) == 6100


@pytest.mark.parametrize("N,bound", [(1, "hbm"), (2, "hbm"), (3, "tensor"), (4, "tensor"), (5, "tensor"), (6, "tensor")])
def test_binding_roofline_by_order(N, bound):
    """HBM binds at N <= 2 (N = 1: 3.4 flop/B against a ridge of 37.04 / 6.55 = 5.7), FP64 from
    N = 3 up; frac is the binding fraction, both fractions are reported and frac is their max."""
    r = bench.roofline(bench.flops_per_elem_stage(N), bench.bytes_per_elem_stage(N), 1_000_000, 1.0, None)
    assert r["bound"] == bound
    assert r["unit"] == ("GB/s" if bound == "hbm" else "TFLOP/s")
    assert r["frac"] == max(r["fp64_frac"], r["hbm_frac"])
    assert abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-3


def test_roofline_numbers_of_a_known_line():
    # the round-2 C4 line: 1,473,114 elements in 4.58 ms per stage -> 22.4 TFLOP/s, 0.605 of 37.04
    r = bench.roofline(69675, 5824, 1473114, 4.58, 9.77e9)
    assert r["bound"] == "tensor" and abs(r["achieved"] - 22.41) < 0.02 and abs(r["frac"] - 0.605) < 1e-3
    assert r["traffic"] == 9.77e9 and r["peak"] == bench.FP64_PEAK_TFLOPS
