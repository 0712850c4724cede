// filter_gpu.cpp -- the binding of INTEGRATION.md section 1: the reference's
// fbf::fast_bilateral (include/fourierbf/filter.hpp:43-46) on a B200 through
// libfbf.so's C ABI (include/fbf.h). A maintainer adds this file to the
// reference's src/ and links libfbf.so; tests/integration/integration_main.cpp
// compiles it against the reference's own headers and checks it against the
// reference's fast_bilateral (oracle/Makefile target `integration`).
#include <stdexcept>
#include <vector>

#include "fourierbf/filter.hpp"
extern "C" {
#include "fbf.h"
}

namespace fbf {

// Same signature and semantics as fast_bilateral; `threads` has no meaning on
// the GPU. Exceptions as in filter.cpp: std::invalid_argument for a malformed
// approximation (:132-134) and out-of-range pixels (:19-23).
GrayImage fast_bilateral_gpu(const GrayImage& img, const SpatialKernel& kernel, const FourierApproximation& approx,
                             BorderPolicy border, FilterDiagnostics* diag = nullptr, int /*threads*/ = 1,
                             StageTimings* timings = nullptr) {
    if (approx.terms < 1 || approx.coefficients.size() != static_cast<size_t>(approx.terms))
        throw std::invalid_argument("fast_bilateral: malformed approximation");
    std::vector<float> in(img.pixels.begin(), img.pixels.end()), out(in.size());
    long long fallbacks = 0;
    fbf_stage_timings st{};
    const int rc = fbf_fast_bilateral_ex(in.data(), img.width, img.height, kernel.theta, approx.terms,
                                         approx.half_period, approx.dynamic_range, approx.frequency,
                                         approx.coefficients.data(), static_cast<int>(border), out.data(),
                                         &fallbacks, timings ? &st : nullptr);
    if (rc == FBF_EINVAL || rc == FBF_ERANGE) throw std::invalid_argument(fbf_last_error());
    if (rc != FBF_OK) throw std::runtime_error(fbf_last_error());
    if (diag) diag->fallback_pixels += fallbacks;
    if (timings) {
        timings->auxiliary_seconds += st.auxiliary_seconds;
        timings->convolution_seconds += st.convolution_seconds;
        timings->combine_seconds += st.combine_seconds;
    }
    GrayImage res(img.width, img.height);
    res.pixels.assign(out.begin(), out.end());
    return res;
}

}  // namespace fbf
