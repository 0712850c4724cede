"""Host parameter selection (libfbf.so, C++ restatement of approx.cpp without
Eigen) pinned to the reference's frozen values and cross-checked against the
numpy oracle. CPU only: these entry points never touch the GPU."""
import numpy as np
import pytest

from oracle import fbf_oracle as fo


def gauss(fb, sigma, R=255):
    return fb.sample_range_kernel(fb.RangeKernelSpec.gaussian(sigma, R))


def test_range_kernel_samples_match_oracle(fb, oracle):
    for kind, sigma in (("gaussian", 50.0), ("exponential", 30.0), ("cauchy", 20.0)):
        spec = getattr(fb.RangeKernelSpec, kind)(sigma, 255)
        assert np.array_equal(fb.sample_range_kernel(spec).values, oracle.range_samples(kind, sigma))
    with pytest.raises(fb.InvalidArgument):
        fb.sample_range_kernel(fb.RangeKernelSpec.gaussian(0.0))


def test_spatial_kernel_matches_oracle(fb, oracle):
    for theta in (0.5, 1.0, 3.0, 5.0, 10.0):
        k = fb.build_spatial_kernel(theta)
        assert k.radius == int(np.ceil(3 * theta))
        assert np.array_equal(k.taps, oracle.spatial_taps(theta))
    with pytest.raises(fb.InvalidArgument):
        fb.build_spatial_kernel(-1.0)


def test_frozen_error_sigma50_K4_T203(fb):
    # test_approx.cpp:73-93
    assert fb.fit_error(gauss(fb, 50.0), 4, 203) == pytest.approx(0.0096065911564679699, rel=1e-8)


def test_fit_agrees_with_numpy_lstsq(fb, oracle):
    for sigma, K, T in ((50.0, 4, 203), (30.0, 5, 168), (15.0, 9, 150), (80.0, 3, 239), (40.0, 4, 255)):
        b = oracle.range_samples("gaussian", sigma)
        c_ref, e_ref = fo.fit_coefficients(fo.design_matrix(K, T, 255), b)
        a = fb.fit_fixed_period(fb.sample_range_kernel(fb.RangeKernelSpec.gaussian(sigma)), K, T)
        assert np.allclose(a.coefficients, c_ref, rtol=1e-8, atol=1e-12)
        assert fb.fit_error(fb.sample_range_kernel(fb.RangeKernelSpec.gaussian(sigma)), K, T) == pytest.approx(e_ref, rel=1e-8)


def test_optimal_period_and_tie_break(fb):
    assert fb.min_error_over_period(4, gauss(fb, 50.0), 400).best_half_period == 203   # :102-107
    b = gauss(fb, 25.0)
    assert fb.min_error_over_period(1, b, 60).best_half_period == 1                    # :109-116
    e = fb.scan_period_errors(1, b, 60)
    assert np.all(e == e[0])


def test_sigma40_period_and_fbf_baseline(fb):
    # test_approx.cpp:211-227
    b = gauss(fb, 40.0)
    scan = fb.min_error_over_period(4, b, 500)
    assert scan.best_half_period == 179
    assert scan.best_error == pytest.approx(0.039303651041756635, rel=1e-6)
    assert fb.fit_error(b, 4, 255) == pytest.approx(0.92015684935042141, rel=1e-6)
    # the CLI's default T_max = 10 R gives the same period (tests/CMakeLists.txt:45-50)
    assert fb.select_parameters(40.0, K=4).half_period == 179


def test_algorithm1_sigma50_eps01(fb):
    # test_approx.cpp:124-136, acceptance.cpp:71-90 (default T_max)
    rep = fb.optimize_parameters(gauss(fb, 50.0), 0.1, fb.OptimizeOptions(t_max=400))
    assert (rep.best_terms, rep.best_half_period) == (4, 203)
    assert len(rep.per_order) == 4
    assert all(rep.per_order[i].best_error <= rep.per_order[i - 1].best_error + 1e-10 for i in range(1, 4))
    rep = fb.optimize_parameters(gauss(fb, 50.0), 0.1, fb.OptimizeOptions(threads=8))
    assert (rep.best_terms, rep.best_half_period) == (4, 203)


def test_full_order_vanishes_toy_R7(fb):
    # test_approx.cpp:118-122, 146-151
    b = gauss(fb, 1.0, 7)
    assert fb.min_error_over_period(15, b, 70).best_error <= 1e-10
    rep = fb.optimize_parameters(b, 1e-12)
    assert rep.best_terms <= 15 and rep.achieved_error <= 1e-12


def test_constant_kernel_needs_one_term(fb):
    b = fb.tabulated_samples(np.ones(31))
    rep = fb.optimize_parameters(b, 1e-6)
    assert rep.best_terms == 1 and rep.achieved_error <= 1e-24


def test_tolerance_unreachable(fb):
    # test_approx.cpp:153-181
    with pytest.raises(fb.ToleranceUnreachable) as e:
        fb.optimize_parameters(gauss(fb, 50.0), 0.1, fb.OptimizeOptions(t_max=3))
    assert "saturates" in str(e.value)
    assert len(e.value.best_found.per_order) <= 4 and e.value.best_found.achieved_error > 0.1
    with pytest.raises(fb.ToleranceUnreachable) as e:
        fb.optimize_parameters(gauss(fb, 50.0), 1e-9, fb.OptimizeOptions(t_max=400, k_max=3))
    bf = e.value.best_found
    assert len(bf.per_order) == 3 and bf.best_terms == 3 and len(bf.coefficients) == 3 and bf.achieved_error > 1e-9


def test_select_parameters_cli_semantics(fb):
    # tools/fourierbf.cpp:185-234
    a = fb.select_parameters(50.0, K=4, T=203)
    assert (a.terms, a.half_period) == (4, 203)
    a = fb.select_parameters(50.0, K=4, method="fbf")
    assert a.half_period == 255
    a = fb.select_parameters(50.0, eps=0.1, method="fbf")
    assert (a.terms, a.half_period) == (4, 255)
    with pytest.raises(fb.InvalidArgument):
        fb.select_parameters(50.0, eps=0.1, K=4)
    with pytest.raises(fb.InvalidArgument):
        fb.select_parameters(50.0, T=100)
    with pytest.raises(fb.InvalidArgument):
        fb.select_parameters(50.0)


def test_baseline_config_parameters(fb):
    # (K, T) chosen by the reference algorithm per config
    from paper_1811_02168_b200 import configs
    for name, cfg in configs.CONFIGS.items():
        a = configs.select(cfg)
        assert (a.terms, a.half_period) == cfg.expect_KT, name


def test_approximation_evaluate_and_tabulate(fb, oracle):
    a = fb.fit_fixed_period(gauss(fb, 50.0), 4, 203)
    assert a.evaluate(0) == pytest.approx(sum(a.coefficients), rel=1e-15)
    tab = fb.tabulate_approximation(a)
    assert np.array_equal(tab.values, oracle.tabulate(4, 203, 255, a.coefficients))
