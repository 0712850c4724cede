// integration_main.cpp -- TEST: the INTEGRATION.md section 1 binding
// (filter_gpu.cpp) compiled against the reference's own headers and linked with
// the reference's filter.cpp / kernels.cpp / synthetic.cpp and libfbf.so. Runs
// the reference fast_bilateral and the GPU binding on the reference's own
// random_image / scene_image inputs with identical (K, T, c) and checks the
// contract: max |gpu - ref| <= 1e-2, equal fallback counts, the same exception
// classes (test_filter.cpp:168-183, 240-268). Exit 0 and "INTEGRATION OK" on success.
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "fourierbf/filter.hpp"
#include "fourierbf/synthetic.hpp"
extern "C" {
#include "fbf.h"
}

namespace fbf {
GrayImage fast_bilateral_gpu(const GrayImage& img, const SpatialKernel& kernel, const FourierApproximation& approx,
                             BorderPolicy border, FilterDiagnostics* diag = nullptr, int threads = 1,
                             StageTimings* timings = nullptr);
}

namespace {

int failures = 0;
#define CHECK(cond, ...)                                   \
    do {                                                   \
        if (!(cond)) {                                     \
            std::printf("FAIL %s:%d: ", __FILE__, __LINE__); \
            std::printf(__VA_ARGS__);                      \
            std::printf("\n");                             \
            ++failures;                                    \
        }                                                  \
    } while (0)

// The approximation the reference CLI would pick (select_parameters through
// libfbf's Eigen-free restatement of approx.cpp).
fbf::FourierApproximation select(double sigma, double eps, int K) {
    std::vector<double> c(511);
    int Ko = 0, To = 0;
    double err = 0;
    if (fbf_select_params(FBF_KERNEL_GAUSSIAN, sigma, 255, eps, K, 0, 0, 8, &Ko, &To, c.data(), 511, &err) != FBF_OK)
        throw std::runtime_error(fbf_last_error());
    fbf::FourierApproximation a;
    a.terms = Ko;
    a.half_period = To;
    a.dynamic_range = 255;
    a.frequency = 2.0 * 3.14159265358979323846 / (2.0 * To + 1.0);
    a.coefficients.assign(c.begin(), c.begin() + Ko);
    return a;
}

double max_abs(const fbf::GrayImage& a, const fbf::GrayImage& b) {
    double m = 0;
    for (size_t i = 0; i < a.pixels.size(); ++i) m = std::fmax(m, std::fabs(a.pixels[i] - b.pixels[i]));
    return m;
}

}  // namespace

int main() {
    double worst = 0;
    const fbf::BorderPolicy borders[] = {fbf::BorderPolicy::symmetric, fbf::BorderPolicy::replicate,
                                         fbf::BorderPolicy::zero};
    struct Case {
        int w, h;
        double theta, sigma, eps;
        int K;
    } cases[] = {{64, 48, 3.0, 30.0, 0.1, 0}, {97, 61, 5.0, 50.0, 0.0, 4}, {40, 35, 8.0, 15.0, 0.01, 0},
                 {300, 200, 10.0, 80.0, 0.05, 0}};
    int n = 0;
    for (const Case& cs : cases) {
        const auto approx = select(cs.sigma, cs.eps, cs.K);
        const auto kernel = fbf::build_spatial_kernel(cs.theta);
        for (int s = 0; s < 2; ++s) {
            const auto img = s == 0 ? fbf::random_image(cs.w, cs.h, 17 + n) : fbf::scene_image(cs.w, cs.h, 29 + n);
            for (auto border : borders) {
                fbf::FilterDiagnostics d_ref, d_gpu;
                const auto ref = fbf::fast_bilateral(img, kernel, approx, border, &d_ref, 4);
                const auto gpu = fbf::fast_bilateral_gpu(img, kernel, approx, border, &d_gpu);
                const double e = max_abs(ref, gpu);
                worst = std::fmax(worst, e);
                CHECK(e <= 1e-2, "case %d border %d: max |gpu - ref| = %g", n, (int)border, e);
                CHECK(d_ref.fallback_pixels == d_gpu.fallback_pixels, "fallbacks %lld vs %lld",
                      d_ref.fallback_pixels, d_gpu.fallback_pixels);
            }
            ++n;
        }
    }
    // all-zero coefficients: every pixel falls back to its input (test_filter.cpp:240-268)
    {
        auto approx = select(30.0, 0.1, 0);
        for (double& c : approx.coefficients) c = 0.0;
        const auto img = fbf::random_image(6, 6, 3);
        fbf::FilterDiagnostics d_ref, d_gpu;
        const auto ref = fbf::fast_bilateral(img, fbf::build_spatial_kernel(2.0), approx,
                                             fbf::BorderPolicy::symmetric, &d_ref);
        const auto gpu = fbf::fast_bilateral_gpu(img, fbf::build_spatial_kernel(2.0), approx,
                                                 fbf::BorderPolicy::symmetric, &d_gpu);
        CHECK(d_ref.fallback_pixels == 36 && d_gpu.fallback_pixels == 36, "fallbacks %lld / %lld",
              d_ref.fallback_pixels, d_gpu.fallback_pixels);
        CHECK(max_abs(gpu, img) == 0.0, "fallback output must be the input");
    }
    // exception classes (filter.cpp:19-23, 132-134)
    {
        const auto approx = select(30.0, 0.1, 0);
        auto img = fbf::random_image(16, 16, 5);
        img.at(3, 4) = 300.0;
        bool ref_threw = false, gpu_threw = false;
        try { fbf::fast_bilateral(img, fbf::build_spatial_kernel(2.0), approx, fbf::BorderPolicy::symmetric); }
        catch (const std::invalid_argument&) { ref_threw = true; }
        try { fbf::fast_bilateral_gpu(img, fbf::build_spatial_kernel(2.0), approx, fbf::BorderPolicy::symmetric); }
        catch (const std::invalid_argument&) { gpu_threw = true; }
        CHECK(ref_threw && gpu_threw, "pixel range: invalid_argument ref %d gpu %d", ref_threw, gpu_threw);
        auto bad = approx;
        bad.coefficients.pop_back();
        ref_threw = gpu_threw = false;
        const auto ok = fbf::random_image(8, 8, 6);
        try { fbf::fast_bilateral(ok, fbf::build_spatial_kernel(2.0), bad, fbf::BorderPolicy::symmetric); }
        catch (const std::invalid_argument&) { ref_threw = true; }
        try { fbf::fast_bilateral_gpu(ok, fbf::build_spatial_kernel(2.0), bad, fbf::BorderPolicy::symmetric); }
        catch (const std::invalid_argument&) { gpu_threw = true; }
        CHECK(ref_threw && gpu_threw, "malformed approx: invalid_argument ref %d gpu %d", ref_threw, gpu_threw);
    }
    // StageTimings are filled by accumulation
    {
        const auto approx = select(50.0, 0.0, 4);
        fbf::StageTimings t;
        fbf::fast_bilateral_gpu(fbf::random_image(512, 512, 9), fbf::build_spatial_kernel(5.0), approx,
                                fbf::BorderPolicy::symmetric, nullptr, 1, &t);
        CHECK(t.convolution_seconds > 0.0, "StageTimings::convolution_seconds = %g", t.convolution_seconds);
    }
    if (failures) {
        std::printf("INTEGRATION FAILED (%d checks)\n", failures);
        return 1;
    }
    std::printf("INTEGRATION OK cases=%d max_abs_gpu_minus_reference=%.3e\n", n * 3, worst);
    return 0;
}
