// ref_bridge.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the reference's OWN fourierbf sources
// (filter.cpp, kernels.cpp, synthetic.cpp compiled verbatim from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libfbf_ref.so).
// This is the strongest oracle available: the reference's fast_bilateral run on
// the same (float32 -> double widened) pixels with the same (K, T, c).
// Used by tests/ to pin oracle/fbf_oracle.c and by bench.py --impl reference.
#include <cmath>
#include <exception>
#include <numbers>
#include <vector>

#include "fourierbf/filter.hpp"
#include "fourierbf/kernels.hpp"
#include "fourierbf/synthetic.hpp"

namespace {

fbf::BorderPolicy border_of(int b) {
    return b == 1 ? fbf::BorderPolicy::replicate
                  : (b == 2 ? fbf::BorderPolicy::zero : fbf::BorderPolicy::symmetric);
}

// approx.cpp:17-19 restated (approx.cpp itself needs Eigen).
double frequency_of(int half_period) {
    return 2.0 * std::numbers::pi / (2.0 * half_period + 1.0);
}

fbf::GrayImage wrap(const double* img, int w, int h) {
    fbf::GrayImage g(w, h);
    for (size_t i = 0; i < g.pixels.size(); ++i) g.pixels[i] = img[i];
    return g;
}

}  // namespace

extern "C" {

int fbfref_fast_bilateral(const double* img, int w, int h, double theta, int K, int T, int R,
                          const double* coeffs, int border, int threads, double* out,
                          long long* fallbacks, double* stage_seconds) {
    try {
        fbf::FourierApproximation a;
        a.terms = K;
        a.half_period = T;
        a.dynamic_range = R;
        a.frequency = frequency_of(T);
        a.coefficients.assign(coeffs, coeffs + K);
        const auto kernel = fbf::build_spatial_kernel(theta);
        fbf::FilterDiagnostics diag;
        fbf::StageTimings st;
        const auto res = fbf::fast_bilateral(wrap(img, w, h), kernel, a, border_of(border), &diag,
                                             threads, &st);
        for (size_t i = 0; i < res.pixels.size(); ++i) out[i] = res.pixels[i];
        if (fallbacks) *fallbacks += diag.fallback_pixels;
        if (stage_seconds) {
            stage_seconds[0] = st.auxiliary_seconds;
            stage_seconds[1] = st.convolution_seconds;
            stage_seconds[2] = st.combine_seconds;
        }
        return 0;
    } catch (const std::invalid_argument&) {
        return -2;
    } catch (...) {
        return -1;
    }
}

int fbfref_brute_bilateral(const double* img, int w, int h, double theta, const double* range,
                           int R, int border, int threads, double* out, long long* fallbacks) {
    try {
        fbf::RangeKernelSamples s;
        s.dynamic_range = R;
        s.values.assign(range, range + 2 * R + 1);
        const auto kernel = fbf::build_spatial_kernel(theta);
        fbf::FilterDiagnostics diag;
        const auto res =
            fbf::brute_bilateral(wrap(img, w, h), kernel, s, border_of(border), &diag, threads);
        for (size_t i = 0; i < res.pixels.size(); ++i) out[i] = res.pixels[i];
        if (fallbacks) *fallbacks += diag.fallback_pixels;
        return 0;
    } catch (const std::invalid_argument&) {
        return -2;
    } catch (...) {
        return -1;
    }
}

int fbfref_convolve_separable(const double* img, int w, int h, double theta, int border,
                              double* out) {
    try {
        const auto kernel = fbf::build_spatial_kernel(theta);
        const auto res = fbf::convolve_separable(wrap(img, w, h), kernel, border_of(border), 1);
        for (size_t i = 0; i < res.pixels.size(); ++i) out[i] = res.pixels[i];
        return 0;
    } catch (...) {
        return -1;
    }
}

int fbfref_spatial_taps(double theta, double* taps) {
    const auto k = fbf::build_spatial_kernel(theta);
    for (size_t i = 0; i < k.taps.size(); ++i) taps[i] = k.taps[i];
    return k.radius;
}

int fbfref_range_samples(int kind, double sigma, int R, double* values) {
    try {
        fbf::RangeKernelSpec spec = kind == 1   ? fbf::RangeKernelSpec::exponential(sigma, R)
                                    : kind == 2 ? fbf::RangeKernelSpec::cauchy(sigma, R)
                                                : fbf::RangeKernelSpec::gaussian(sigma, R);
        const auto s = fbf::sample_range_kernel(spec);
        for (size_t i = 0; i < s.values.size(); ++i) values[i] = s.values[i];
        return 0;
    } catch (...) {
        return -1;
    }
}

void fbfref_random_image(int w, int h, unsigned long long seed, double* out) {
    const auto g = fbf::random_image(w, h, seed);
    for (size_t i = 0; i < g.pixels.size(); ++i) out[i] = g.pixels[i];
}

void fbfref_scene_image(int w, int h, unsigned long long seed, double* out) {
    const auto g = fbf::scene_image(w, h, seed);
    for (size_t i = 0; i < g.pixels.size(); ++i) out[i] = g.pixels[i];
}

}  // extern "C"
