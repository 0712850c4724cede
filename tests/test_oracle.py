"""The CPU oracle (oracle/fbf_oracle.c + numpy optimiser) pinned against the reference.

Golden fixtures (tests/golden/reference_golden.npz) were produced by the
reference's own sources compiled verbatim (tests/golden/make_golden.py); the C
restatement must reproduce them bit for bit. When the reference build is
present, random cases are compared live as well.
"""
import numpy as np
import pytest

from oracle import fbf_oracle as fo


def test_spatial_taps_and_range_samples(oracle, golden):
    for theta in (1.0, 2.0, 3.0, 5.0, 8.0, 10.0):
        assert np.array_equal(oracle.spatial_taps(theta), golden[f"taps_theta{theta:g}"])
    for kind, sigma in (("gaussian", 50.0), ("gaussian", 15.0), ("exponential", 30.0), ("cauchy", 20.0)):
        assert np.array_equal(oracle.range_samples(kind, sigma), golden[f"range_{kind}_{sigma:g}"])


def test_synthetic_images(oracle, golden):
    assert np.array_equal(oracle.random_image(24, 24, 7000), golden["random_24x24_7000"])
    assert np.array_equal(oracle.random_image(5, 4, 7), golden["random_5x4_7"])
    assert np.array_equal(oracle.scene_image(96, 96, 2024), golden["scene_96x96_2024"])


def test_fast_bilateral_bit_exact_against_reference_golden(oracle, golden):
    cases = [c for c in open(fo.HERE + "/../tests/golden/cases.txt").read().split() if c]
    assert len(cases) == 27
    for key in cases:
        K, T = golden[key + "_KT"]
        border = key.rsplit("_", 1)[1]
        theta = float(key.split("_t")[1].split("_")[0])
        out, fb = oracle.fast_bilateral(golden[key + "_img"], theta, int(K), int(T), golden[key + "_coeffs"],
                                        border=border)
        assert fb == 0
        assert np.array_equal(out, golden[key + "_out"]), key


def test_radius_wider_than_image(oracle, golden):
    # test_filter.cpp:73-81: radius 9 > both dimensions of a 5x4 image
    img = golden["random_5x4_7"]
    for border in ("symmetric", "replicate", "zero"):
        out, _ = oracle.fast_bilateral(img, 3.0, 4, 203, golden["c_sigma50_K4_T203"], border=border)
        assert np.array_equal(out, golden[f"fast_5x4_{border}_out"])


def test_brute_scene_golden(oracle, golden):
    out, _ = oracle.brute_bilateral(golden["scene_96x96_2024"], 5.0, oracle.range_samples("gaussian", 55.0))
    assert np.array_equal(out, golden["brute_scene96_t5_s55"])


def test_map_border_index_matches_step_folding(oracle):
    # tests/oracles.hpp:112-124 folds step by step; image.hpp uses modular folding
    def fold(i, n, border):
        if border == 2:
            return -1 if (i < 0 or i >= n) else i
        if border == 1:
            return 0 if i < 0 else (n - 1 if i >= n else i)
        while i < 0 or i >= n:
            if i < 0:
                i = -i - 1
            if i >= n:
                i = 2 * n - 1 - i
        return i
    for n in (1, 2, 3, 5, 8):
        for i in range(-25, 30):
            for border in range(3):
                assert oracle.map_border_index(i, n, border) == fold(i, n, border)


def test_constant_and_impulse_convolution(oracle):
    # test_filter.cpp:33-61
    taps = oracle.spatial_taps(2.0)
    s = taps.sum()
    img = np.full((15, 20), 3.25)
    for border in ("symmetric", "replicate"):
        out = oracle.convolve_separable(img, 2.0, border)
        assert np.allclose(out, 3.25 * s * s, rtol=1e-12)
    out = oracle.convolve_separable(img, 2.0, "zero")
    assert out[7, 10] == pytest.approx(3.25 * s * s, rel=1e-12) and out[0, 0] < 3.25 * s * s
    imp = np.zeros((15, 15))
    imp[7, 7] = 1.0
    t1 = oracle.spatial_taps(1.0)
    out = oracle.convolve_separable(imp, 1.0, "zero")
    assert np.allclose(out[4:11, 4:11], np.outer(t1, t1), rtol=1e-14)


def test_fast_equals_brute_with_substituted_kernel(oracle):
    # test_filter.cpp:156-166 (integer image, 1e-6)
    img = oracle.random_image(32, 32, 1234)
    b = oracle.range_samples("gaussian", 50.0)
    rep = fo.optimize_parameters(b, 0.1, t_max=500)
    table = oracle.tabulate(rep.K, rep.T, 255, rep.coefficients)
    for border in ("symmetric", "replicate", "zero"):
        fast, _ = oracle.fast_bilateral(img, 3.0, rep.K, rep.T, rep.coefficients, border=border)
        brute, _ = oracle.brute_bilateral(img, 3.0, table, border=border)
        assert np.abs(fast - brute).max() <= 1e-6


def test_optimizer_restatement_pins():
    o = fo.Oracle()
    b50 = o.range_samples("gaussian", 50.0)
    c, e = fo.fit_coefficients(fo.design_matrix(4, 203, 255), b50)
    assert e == pytest.approx(0.0096065911564679699, rel=1e-8)          # test_approx.cpp:86
    assert fo.min_error_over_period(4, b50, 400)[0] == 203             # test_approx.cpp:105
    rep = fo.optimize_parameters(b50, 0.1, t_max=400)
    assert (rep.K, rep.T) == (4, 203)                                   # test_approx.cpp:129-130
    b40 = o.range_samples("gaussian", 40.0)
    T, e40 = fo.min_error_over_period(4, b40, 500)
    assert T == 179 and e40 == pytest.approx(0.039303651041756635, rel=1e-6)  # :223-224
    assert fo.fit_coefficients(fo.design_matrix(4, 255, 255), b40)[1] == pytest.approx(0.92015684935042141, rel=1e-6)
    errs = fo.scan_period_errors(1, o.range_samples("gaussian", 25.0), 60)  # :109-116
    assert np.all(errs == errs[0])


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_oracle_matches_reference_live(oracle, ref_lib, seed):
    rng = np.random.default_rng(seed)
    h, w = rng.integers(3, 40, size=2)
    img = rng.uniform(0, 255, size=(h, w))
    theta = float(rng.choice([0.7, 1.0, 2.5, 4.0]))
    K = int(rng.integers(1, 6))
    c = rng.normal(size=K)
    for border in ("symmetric", "replicate", "zero"):
        a, fa = oracle.fast_bilateral(img, theta, K, 150, c, border=border)
        b, fb_ = ref_lib.fast_bilateral(img, theta, K, 150, c, border=border)
        assert np.array_equal(a, b) and fa == fb_
