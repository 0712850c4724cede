// fbf_synth.cpp -- synthetic inputs.
//
// random_image / scene_image restate the reference's synthetic module
// (/root/reference/proj/src/synthetic.cpp:9-64) in float32. The Voronoi and
// sinusoid-field generators are NEW: BASELINE.json's five configs name them
// but the reference has none. They stand in for the
// paper's public evaluation images, which are not available here. All draws
// come from the reference's SplitMix64; per-row noise streams are seeded
// independently so the images are identical for every thread count.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <numbers>
#include <vector>

#include "../../include/fbf.h"
#include "fbf_internal.h"

namespace {

// synthetic.cpp:9-21
struct SplitMix64 {
    uint64_t state;
    explicit SplitMix64(uint64_t seed) : state(seed) {}
    uint64_t next() {
        uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    // Box-Muller (one deviate per two uniforms); 1-u keeps log() finite
    double normal() {
        const double u1 = uniform(), u2 = uniform();
        return std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(2.0 * std::numbers::pi * u2);
    }
};

uint64_t row_stream_seed(uint64_t seed, int y) {
    return seed ^ (0xd1b54a32d192ed03ULL * static_cast<uint64_t>(y + 1));
}

struct Sites {
    int n = 0;
    std::vector<double> x, y, v;
    // uniform bucket grid for nearest-site queries
    int gx = 1, gy = 1;
    double cw = 1, ch = 1;
    std::vector<std::vector<int>> cells;

    Sites(int width, int height, int count, SplitMix64& rng, double vlo, double vhi) : n(count) {
        x.resize(n);
        y.resize(n);
        v.resize(n);
        for (int i = 0; i < n; ++i) {
            x[i] = rng.uniform() * width;
            y[i] = rng.uniform() * height;
            v[i] = vlo + (vhi - vlo) * rng.uniform();
        }
        const double side = std::sqrt(static_cast<double>(width) * height / std::max(1, n));
        gx = std::max(1, static_cast<int>(width / side));
        gy = std::max(1, static_cast<int>(height / side));
        cw = static_cast<double>(width) / gx;
        ch = static_cast<double>(height) / gy;
        cells.assign(static_cast<size_t>(gx) * gy, {});
        for (int i = 0; i < n; ++i) {
            const int cx = std::min(gx - 1, static_cast<int>(x[i] / cw));
            const int cy = std::min(gy - 1, static_cast<int>(y[i] / ch));
            cells[static_cast<size_t>(cy) * gx + cx].push_back(i);
        }
    }

    // nearest site to (px, py) by squared distance; ties -> lowest index
    int nearest(double px, double py) const {
        const int cx = std::min(gx - 1, static_cast<int>(px / cw));
        const int cy = std::min(gy - 1, static_cast<int>(py / ch));
        double best = std::numeric_limits<double>::infinity();
        int bi = -1;
        const double step = std::min(cw, ch);
        for (int ring = 0;; ++ring) {
            for (int yy = cy - ring; yy <= cy + ring; ++yy) {
                if (yy < 0 || yy >= gy) continue;
                for (int xx = cx - ring; xx <= cx + ring; ++xx) {
                    if (xx < 0 || xx >= gx) continue;
                    if (std::max(std::abs(xx - cx), std::abs(yy - cy)) != ring) continue;
                    for (int i : cells[static_cast<size_t>(yy) * gx + xx]) {
                        const double dx = x[i] - px, dy = y[i] - py;
                        const double d = dx * dx + dy * dy;
                        if (d < best || (d == best && i < bi)) {
                            best = d;
                            bi = i;
                        }
                    }
                }
            }
            // any site beyond this ring is at least ring*step away
            const double reach = ring * step;
            if (bi >= 0 && best < reach * reach) break;
            if (ring > gx + gy) break;
        }
        return bi;
    }
};

float clip255(double v) { return static_cast<float>(std::min(255.0, std::max(0.0, v))); }

}  // namespace

extern "C" {

void fbf_random_image_f32(int width, int height, unsigned long long seed, float* out) {
    SplitMix64 rng(seed);  // synthetic.cpp:25-31
    const size_t n = static_cast<size_t>(width) * height;
    for (size_t i = 0; i < n; ++i) out[i] = static_cast<float>(rng.next() % 256);
}

void fbf_scene_image_f32(int width, int height, unsigned long long seed, float* out) {
    SplitMix64 rng(seed);  // synthetic.cpp:33-64
    const double cx = 0.35 * width, cy = 0.4 * height;
    const double disk_r = 0.22 * std::min(width, height);
    const double rx0 = 0.55 * width, ry0 = 0.55 * height;
    const double rx1 = 0.9 * width, ry1 = 0.85 * height;
    for (int y = 0; y < height; ++y)
        for (int x = 0; x < width; ++x) {
            double v = 40.0 + 120.0 * (static_cast<double>(x) / width) +
                       25.0 * std::sin(6.0 * static_cast<double>(y) / height);
            const double dx = x - cx, dy = y - cy;
            if (dx * dx + dy * dy < disk_r * disk_r) v = 220.0;
            if (x >= rx0 && x <= rx1 && y >= ry0 && y <= ry1) v = 30.0;
            if (x - y > 0.55 * width) v = 170.0;
            v += (rng.uniform() - 0.5) * 8.0;
            v = std::round(v);
            out[static_cast<size_t>(y) * width + x] =
                static_cast<float>(std::min(255.0, std::max(0.0, v)));
        }
}

void fbf_voronoi_image_f32(int width, int height, int n_sites, double noise,
                           unsigned long long seed, int threads, float* out) {
    SplitMix64 rng(seed);
    const Sites s(width, height, std::max(1, n_sites), rng, 0.0, 255.0);
    fbf_b200::parallel_for(0, height, threads, [&](int y) {
        SplitMix64 nr(row_stream_seed(seed, y));
        float* row = out + static_cast<size_t>(y) * width;
        for (int x = 0; x < width; ++x) {
            const int i = s.nearest(x + 0.5, y + 0.5);
            row[x] = clip255(s.v[i] + noise * nr.normal());
        }
    });
}

void fbf_field_image_f32(int width, int height, int n_sites, double noise,
                         unsigned long long seed, int threads, float* out) {
    constexpr int kWaves = 32;
    SplitMix64 rng(seed);
    double u[kWaves], v[kWaves], a[kWaves], ph[kWaves];
    for (int i = 0; i < kWaves; ++i) {
        u[i] = 1.0 + 7.0 * rng.uniform();  // cycles across the width
        v[i] = 1.0 + 7.0 * rng.uniform();  // cycles across the height
        a[i] = 0.5 + 0.5 * rng.uniform();
        ph[i] = 2.0 * std::numbers::pi * rng.uniform();
    }
    const Sites s(width, height, std::max(1, n_sites), rng, -64.0, 64.0);
    // sin(A(x) + B(y)) = sin A cos B + cos A sin B with separable tables
    std::vector<double> sa(static_cast<size_t>(width) * kWaves), ca(sa.size());
    for (int x = 0; x < width; ++x)
        for (int i = 0; i < kWaves; ++i) {
            const double A = 2.0 * std::numbers::pi * u[i] * x / width + ph[i];
            sa[static_cast<size_t>(x) * kWaves + i] = a[i] * std::sin(A);
            ca[static_cast<size_t>(x) * kWaves + i] = a[i] * std::cos(A);
        }
    std::vector<double> rmin(height), rmax(height);
    fbf_b200::parallel_for(0, height, threads, [&](int y) {
        double sb[kWaves], cb[kWaves];
        for (int i = 0; i < kWaves; ++i) {
            const double B = 2.0 * std::numbers::pi * v[i] * y / height;
            sb[i] = std::sin(B);
            cb[i] = std::cos(B);
        }
        float* row = out + static_cast<size_t>(y) * width;
        double lo = std::numeric_limits<double>::infinity(), hi = -lo;
        for (int x = 0; x < width; ++x) {
            const double* sx = &sa[static_cast<size_t>(x) * kWaves];
            const double* cx = &ca[static_cast<size_t>(x) * kWaves];
            double acc = 0.0;
            for (int i = 0; i < kWaves; ++i) acc += sx[i] * cb[i] + cx[i] * sb[i];
            row[x] = static_cast<float>(acc);
            lo = std::min(lo, acc);
            hi = std::max(hi, acc);
        }
        rmin[y] = lo;
        rmax[y] = hi;
    });
    const double lo = *std::min_element(rmin.begin(), rmin.end());
    const double hi = *std::max_element(rmax.begin(), rmax.end());
    const double scale = hi > lo ? 255.0 / (hi - lo) : 0.0;
    fbf_b200::parallel_for(0, height, threads, [&](int y) {
        SplitMix64 nr(row_stream_seed(seed, y));
        float* row = out + static_cast<size_t>(y) * width;
        for (int x = 0; x < width; ++x) {
            const int i = s.nearest(x + 0.5, y + 0.5);
            const double smooth = (row[x] - lo) * scale;
            row[x] = clip255(smooth + s.v[i] + noise * nr.normal());
        }
    });
}

}  // extern "C"
