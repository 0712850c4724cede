"""Lookup table (lut.hpp / lut.cpp): translations of the reference's
tests/test_lut.cpp plus the GPU-scan build (identical cells)."""
import numpy as np
import pytest

from paper_1811_02168_b200 import fbf as F
from paper_1811_02168_b200 import lut as L


def hand_table():
    # test_lut.cpp:17-25
    return L.LookupTable(255, [20.0, 40.0], [1.0, 3.0], [[6, 9], [4, 7]], [[150, 180], [200, 240]])


def test_grid_nodes_unchanged():
    t = hand_table()
    assert L.query_lut(t, 20.0, 0.1) == L.LutQuery(6, 150)
    assert L.query_lut(t, 40.0, 0.001) == L.LutQuery(7, 240)


def test_interpolation_rounding():
    # test_lut.cpp:53-64: K rounds up, T to nearest
    t = hand_table()
    assert L.query_lut(t, 30.0, 0.1) == L.LutQuery(5, 175)
    assert L.query_lut(t, 25.0, 0.1) == L.LutQuery(6, 163)
    for sigma in (20.0, 22.0, 31.5, 39.0, 40.0):
        for eps in (0.1, 0.05, 0.004, 0.001):
            assert 4 <= L.query_lut(t, sigma, eps).terms <= 9


def test_equal_orders_interpolate_to_that_order():
    t = L.LookupTable(255, [20.0, 40.0], [1.0, 3.0], [[5, 5], [5, 5]], [[150, 180], [200, 240]])
    for sigma in (20.0, 27.3, 40.0):
        for eps in (0.1, 0.013, 0.001):
            assert L.query_lut(t, sigma, eps).terms == 5


@pytest.mark.parametrize("sigma,eps", [(19.9, 0.1), (40.1, 0.1), (30.0, 0.11), (30.0, 0.0009), (30.0, 0.0)])
def test_outside_grid_is_range_error(sigma, eps):
    with pytest.raises(L.LutRangeError):
        L.query_lut(hand_table(), sigma, eps)


@pytest.mark.parametrize("sig,eps", [([50.0], [0.1, 0.01]), ([30.0, 50.0], [0.1]), ([30.0, 50.0], [0.1, 0.1]),
                                     ([50.0, 30.0], [0.1, 0.01]), ([-5.0, 30.0], [0.1, 0.01]),
                                     ([30.0, 50.0], [0.1, 1.5])])
def test_build_validation(sig, eps):
    # test_lut.cpp:111-118
    with pytest.raises(F.InvalidArgument):
        L.build_lut(sig, eps, 255, 100)


def test_build_failure_identifies_cell():
    with pytest.raises(F.FbfError, match="LUT build failed at cell.*eps="):
        L.build_lut([1.0, 2.0], [1e-1, 1e-9], 7, 2)


def test_build_fills_nodes_with_optimizer_answer():
    # test_lut.cpp:86-103 (host scans)
    t = L.build_lut([30.0, 50.0], [0.1, 0.05], 255, 450, threads=4)
    assert (t.rows(), t.cols()) == (2, 2)
    assert L.query_lut(t, 50.0, 0.1) == L.LutQuery(4, 203)
    rep = F.optimize_parameters(F.sample_range_kernel(F.RangeKernelSpec.gaussian(30.0)), 0.05,
                                F.OptimizeOptions(t_max=450))
    assert (t.terms[0][1], t.half_period[0][1]) == (rep.best_terms, rep.best_half_period)
    t1 = L.build_lut([20.0, 35.0], [0.1, 0.02], 255, 300, threads=1)
    t4 = L.build_lut([20.0, 35.0], [0.1, 0.02], 255, 300, threads=4)
    assert t1 == t4


def test_save_load_round_trip_and_malformed(tmp_path):
    t = hand_table()
    t.logeps_grid = [1.0, float(np.log10(1 / 0.003))]
    p = tmp_path / "t.lut"
    L.save_lut(t, str(p))
    assert L.load_lut(str(p)) == t
    text = p.read_text()
    assert text.startswith("R 255\nsigma 20 40\nlogeps 1 2.5228787452803374\nK 6 9\n")
    bad = {"T_missing": "R 255\nsigma 20 40\nlogeps 1 3\nK 6 9\nK 4 7\nT 1 2\n",
           "nonint": "R 255\nsigma 20 40\nlogeps 1 3\nK 6 x\nK 4 7\nT 1 2\nT 3 4\n",
           "rowlen": "R 255\nsigma 20 40\nlogeps 1 3\nK 6\nK 4 7\nT 1 2\nT 3 4\n",
           "tag": "Q 255\n"}
    for name, body in bad.items():
        p.write_text(body)
        with pytest.raises(RuntimeError):
            L.load_lut(str(p))
    p.write_text("R 255\nsigma 40 20\nlogeps 1 3\nK 6 9\nK 4 7\nT 1 2\nT 3 4\n")
    with pytest.raises(F.InvalidArgument):
        L.load_lut(str(p))


def test_trend_check_reports():
    t = hand_table()
    assert L.check_monotone_trends(t) == []
    t.terms = [[4, 7], [6, 9]]
    t.half_period = [[200, 240], [150, 180]]
    v = L.check_monotone_trends(t)
    assert len(v) == 4 and v[0].axis == "K"


@pytest.mark.gpu
def test_gpu_build_identical_to_host(gpu):
    sig = [10.0, 25.0, 50.0, 90.0]
    eps = [0.1, 0.03, 0.01]
    h = L.build_lut(sig, eps, 255, 0, threads=8)
    g = L.build_lut(sig, eps, 255, 0, threads=8, device=0)
    assert g == h
