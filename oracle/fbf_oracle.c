/*
 * fbf_oracle.c -- TEST INFRASTRUCTURE ONLY (parity checker, never shipped).
 *
 * Double-precision, single-threaded restatement of the reference fourierbf
 * filtering path. Every function names the reference lines it follows
 * (paths relative to /root/reference/proj). Operation order is kept identical
 * to the reference so that, compiled with -ffp-contract=off like the
 * reference's ISO C++20 build, results match it bit for bit (pinned by
 * tests/test_oracle.py against oracle/_ref/libfbf_ref.so).
 */
#include "fbf_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* image.hpp:43-61 -- whole-sample mirror with repeated folding, clamp, or -1. */
int orc_map_border_index(int i, int n, int border) {
    if (i >= 0 && i < n) return i;
    switch (border) {
    case ORC_ZERO: return -1;
    case ORC_REPLICATE: return i < 0 ? 0 : n - 1;
    case ORC_SYMMETRIC: {
        const int period = 2 * n;
        int m = i % period;
        if (m < 0) m += period;
        return m < n ? m : period - 1 - m;
    }
    }
    return -1;
}

/* kernels.cpp:105-118 -- radius = ceil(3 theta). */
int orc_spatial_radius(double theta) {
    if (!(theta > 0.0) || !isfinite(theta)) return -1;
    return (int)ceil(3.0 * theta);
}

/* kernels.cpp:105-118 -- unnormalised taps exp(-j^2/(2 theta^2)), mirrored. */
int orc_build_spatial_kernel(double theta, double* taps) {
    const int r = orc_spatial_radius(theta);
    if (r < 0) return -1;
    for (int j = 0; j <= r; ++j) {
        const double v = exp(-((double)j * j) / (2.0 * theta * theta));
        taps[r + j] = v;
        taps[r - j] = v;
    }
    return r;
}

/* kernels.cpp:19-32 (evaluate_kind) and :78-103 (sample_range_kernel). */
int orc_sample_range_kernel(int kind, double sigma, int R, double* values) {
    if (!(sigma > 0.0) || !isfinite(sigma) || R < 1) return -1;
    for (int t = 0; t <= R; ++t) {
        const double x = (double)t;
        double v;
        switch (kind) {
        case ORC_GAUSSIAN: v = exp(-(x * x) / (2.0 * sigma * sigma)); break;
        case ORC_EXPONENTIAL: v = exp(-fabs(x) / sigma); break;
        case ORC_CAUCHY: v = 1.0 / (1.0 + (x * x) / (sigma * sigma)); break;
        default: return -1;
        }
        values[R + t] = v;
        values[R - t] = v;
    }
    return 0;
}

/* approx.cpp:17-19 -- nu = 2 pi / (2T + 1). */
double orc_frequency_of(int half_period) {
    return 2.0 * 3.141592653589793238462643383279502884 / (2.0 * half_period + 1.0);
}

/* approx.cpp:34-42 -- sum_k c_k cos(nu |t| k). */
double orc_evaluate_approximation(int K, int T, const double* coeffs, int t) {
    const double base = orc_frequency_of(T) * abs(t);
    double sum = 0.0;
    for (int k = 0; k < K; ++k) sum += coeffs[k] * cos(base * k);
    return sum;
}

/* approx.cpp:48-59 -- lattice table of phihat, mirrored. */
void orc_tabulate_approximation(int K, int T, int R, const double* coeffs, double* values) {
    for (int t = 0; t <= R; ++t) {
        const double v = orc_evaluate_approximation(K, T, coeffs, t);
        values[R + t] = v;
        values[R - t] = v;
    }
}

/* filter.cpp:19-23 */
static int valid_intensities(const double* img, size_t n, int R) {
    for (size_t i = 0; i < n; ++i) {
        const double v = img[i];
        if (!isfinite(v) || v < 0.0 || v > (double)R) return 0;
    }
    return 1;
}

/* filter.cpp:27-49 -- row pass; interior fast path and border path both
 * accumulate taps in ascending order. */
static void convolve_rows(const double* in, int w, int h, const double* taps, int r, int border,
                          double* out) {
    for (int y = 0; y < h; ++y) {
        const double* src = in + (size_t)y * w;
        double* dst = out + (size_t)y * w;
        for (int x = 0; x < w; ++x) {
            double sum = 0.0;
            if (x >= r && x + r < w) {
                for (int d = -r; d <= r; ++d) sum += taps[r + d] * src[x + d];
            } else {
                for (int d = -r; d <= r; ++d) {
                    const int sx = orc_map_border_index(x + d, w, border);
                    if (sx >= 0) sum += taps[r + d] * src[sx];
                }
            }
            dst[x] = sum;
        }
    }
}

/* filter.cpp:52-70 -- column pass, weighted source rows in ascending d. */
static void convolve_cols(const double* in, int w, int h, const double* taps, int r, int border,
                          double* out) {
    for (int y = 0; y < h; ++y) {
        double* dst = out + (size_t)y * w;
        for (int x = 0; x < w; ++x) dst[x] = 0.0;
        for (int d = -r; d <= r; ++d) {
            const int sy = orc_map_border_index(y + d, h, border);
            if (sy < 0) continue;
            const double weight = taps[r + d];
            const double* src = in + (size_t)sy * w;
            for (int x = 0; x < w; ++x) dst[x] += weight * src[x];
        }
    }
}

/* filter.cpp:74-81 */
int orc_convolve_separable(const double* img, int w, int h, const double* taps, int radius,
                           int border, double* out) {
    double* tmp = (double*)malloc(sizeof(double) * (size_t)w * h);
    if (!tmp) return -3;
    convolve_rows(img, w, h, taps, radius, border, tmp);
    convolve_cols(tmp, w, h, taps, radius, border, out);
    free(tmp);
    return 0;
}

/* filter.cpp:129-213 -- the shiftable-convolution bilateral filter. */
int orc_fast_bilateral(const double* img, int w, int h, double theta, int K, int T, int R,
                       const double* coeffs, int border, double* out, long long* fallbacks) {
    if (K < 1 || T < 1) return -1;
    const size_t n = (size_t)w * h;
    if (!valid_intensities(img, n, R)) return -2;
    const int r = orc_spatial_radius(theta);
    if (r < 0) return -1;
    double* taps = (double*)malloc(sizeof(double) * (2 * r + 1));
    orc_build_spatial_kernel(theta, taps);
    const double nu = orc_frequency_of(T);

    double* num = (double*)calloc(n, sizeof(double));
    double* den = (double*)calloc(n, sizeof(double));
    double* cos_img = (double*)malloc(sizeof(double) * n);
    double* sin_img = (double*)malloc(sizeof(double) * n);
    double* cos_f = (double*)malloc(sizeof(double) * n);
    double* sin_f = (double*)malloc(sizeof(double) * n);
    double* g0 = (double*)malloc(sizeof(double) * n);
    double* g1 = (double*)malloc(sizeof(double) * n);
    double* g2 = (double*)malloc(sizeof(double) * n);
    double* g3 = (double*)malloc(sizeof(double) * n);

    for (int k = 0; k < K; ++k) {
        const double ck = coeffs[k];
        if (k == 0) {
            /* filter.cpp:149-161: G(f) and G(1) */
            for (size_t i = 0; i < n; ++i) cos_img[i] = 1.0;
            orc_convolve_separable(img, w, h, taps, r, border, g0);
            orc_convolve_separable(cos_img, w, h, taps, r, border, g1);
            for (size_t i = 0; i < n; ++i) {
                num[i] += ck * g0[i];
                den[i] += ck * g1[i];
            }
            continue;
        }
        /* filter.cpp:164-177: modulated images */
        const double omega = nu * k;
        for (size_t i = 0; i < n; ++i) {
            const double f = img[i];
            const double c = cos(omega * f);
            const double s = sin(omega * f);
            cos_img[i] = c;
            sin_img[i] = s;
            cos_f[i] = c * f;
            sin_f[i] = s * f;
        }
        /* filter.cpp:182-194 */
        orc_convolve_separable(cos_f, w, h, taps, r, border, g0);
        orc_convolve_separable(sin_f, w, h, taps, r, border, g1);
        orc_convolve_separable(cos_img, w, h, taps, r, border, g2);
        orc_convolve_separable(sin_img, w, h, taps, r, border, g3);
        for (size_t i = 0; i < n; ++i) {
            num[i] += ck * (cos_img[i] * g0[i] + sin_img[i] * g1[i]);
            den[i] += ck * (cos_img[i] * g2[i] + sin_img[i] * g3[i]);
        }
    }
    /* filter.cpp:197-211: combine with fallback */
    long long fb = 0;
    for (size_t i = 0; i < n; ++i) {
        if (den[i] > 1e-12) {
            out[i] = num[i] / den[i];
        } else {
            out[i] = img[i];
            ++fb;
        }
    }
    if (fallbacks) *fallbacks += fb;
    free(taps); free(num); free(den); free(cos_img); free(sin_img); free(cos_f); free(sin_f);
    free(g0); free(g1); free(g2); free(g3);
    return 0;
}

/* filter.cpp:83-127 -- windowed bilateral over the (2r+1)^2 window. */
int orc_brute_bilateral(const double* img, int w, int h, double theta, const double* range,
                        int R, int border, double* out, long long* fallbacks) {
    const size_t n = (size_t)w * h;
    if (!valid_intensities(img, n, R)) return -2;
    const int r = orc_spatial_radius(theta);
    if (r < 0) return -1;
    double* taps = (double*)malloc(sizeof(double) * (2 * r + 1));
    orc_build_spatial_kernel(theta, taps);
    long long fb = 0;
    for (int y = 0; y < h; ++y) {
        for (int x = 0; x < w; ++x) {
            const double center = img[(size_t)y * w + x];
            double num = 0.0, den = 0.0;
            for (int dy = -r; dy <= r; ++dy) {
                const int sy = orc_map_border_index(y + dy, h, border);
                if (sy < 0) continue;
                const double wy = taps[r + dy];
                const double* src = img + (size_t)sy * w;
                for (int dx = -r; dx <= r; ++dx) {
                    const int sx = orc_map_border_index(x + dx, w, border);
                    if (sx < 0) continue;
                    const double neighbor = src[sx];
                    const long t = lround(neighbor - center);
                    const double weight = wy * taps[r + dx] * range[t + R];
                    num += weight * neighbor;
                    den += weight;
                }
            }
            if (den > 0.0) {
                out[(size_t)y * w + x] = num / den;
            } else {
                out[(size_t)y * w + x] = center;
                ++fb;
            }
        }
    }
    if (fallbacks) *fallbacks += fb;
    free(taps);
    return 0;
}

/* synthetic.cpp:9-21 -- splitmix64. */
static uint64_t sm64_next(uint64_t* state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
static double sm64_uniform(uint64_t* state) {
    return (double)(sm64_next(state) >> 11) * 0x1.0p-53;
}

/* synthetic.cpp:25-31 */
void orc_random_image(int w, int h, uint64_t seed, double* out) {
    uint64_t s = seed;
    const size_t n = (size_t)w * h;
    for (size_t i = 0; i < n; ++i) out[i] = (double)(sm64_next(&s) % 256);
}

/* synthetic.cpp:33-64 */
void orc_scene_image(int width, int height, uint64_t seed, double* out) {
    uint64_t s = seed;
    const double cx = 0.35 * width, cy = 0.4 * height;
    const double disk_r = 0.22 * (width < height ? width : height);
    const double rx0 = 0.55 * width, ry0 = 0.55 * height;
    const double rx1 = 0.9 * width, ry1 = 0.85 * height;
    for (int y = 0; y < height; ++y) {
        for (int x = 0; x < width; ++x) {
            double v = 40.0 + 120.0 * ((double)x / width) + 25.0 * sin(6.0 * (double)y / height);
            const double dx = x - cx, dy = y - cy;
            if (dx * dx + dy * dy < disk_r * disk_r) v = 220.0;
            if (x >= rx0 && x <= rx1 && y >= ry0 && y <= ry1) v = 30.0;
            if (x - y > 0.55 * width) v = 170.0;
            v += (sm64_uniform(&s) - 0.5) * 8.0;
            v = round(v);
            /* std::min(255.0, std::max(0.0, v)) including its signed-zero behaviour */
            const double m = (0.0 < v) ? v : 0.0;
            out[(size_t)y * width + x] = (m < 255.0) ? m : 255.0;
        }
    }
}
