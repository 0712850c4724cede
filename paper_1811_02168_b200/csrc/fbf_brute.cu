// fbf_brute.cu -- the direct bilateral filter and the image comparison on the GPU.
//
// brute_bilateral (/root/reference/proj/src/filter.cpp:83-127): for every pixel,
//   num = sum_{dy, dx} w(dy) w(dx) phi(lround(f(y+dy, x+dx) - f(y, x))) f(y+dy, x+dx),
//   den = the same sum without the trailing f; out = den > 0 ? num / den : f(y, x)
// over the (2r+1)^2 window, border samples through map_border_index
// (include/fourierbf/image.hpp:43-61, zero border: skipped), with the range
// kernel read from its sampled lattice (RangeKernelSamples::at, kernels.hpp:31).
//
// This is the accuracy oracle of the fast filter at full image sizes (the CPU
// version is O((2r+1)^2) per pixel: hours at the 268-MP config). It computes in
// FP64 with the reference's exact operation sequence -- weight = (w_y * w_x) *
// phi(t), num += weight * f, den += weight, dy outer and dx inner, both
// ascending -- with explicitly rounded multiplies and adds (no FMA
// contraction), so on float32 inputs its output equals the reference's
// compiled brute_bilateral bit for bit.
//
// compare_images (src/metrics.cpp:10-26) on device buffers: per-block partial
// sums of squared differences and maxima of |a - b|, reduced on the host in
// block order (deterministic).
#include <cuda_runtime.h>

#include <cmath>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/fbf.h"
#include "fbf_cuda_util.h"
#include "fbf_internal.h"

namespace fbf_dev {

constexpr int kBX = 32, kBY = 8;            // output tile per CTA
constexpr int kBruteMaxRadius = 64;
constexpr int kRangeSmem = 4096;            // range lattices up to this size live in shared memory
constexpr int kCmpThreads = 256, kCmpBlocks = 1184;

// image.hpp:43-61
__device__ __forceinline__ int border_index(int i, int n, int border) {
    if (i >= 0 && i < n) return i;
    if (border == FBF_BORDER_ZERO) return -1;
    if (border == FBF_BORDER_REPLICATE) return i < 0 ? 0 : n - 1;
    const int period = 2 * n;
    int m = i % period;
    if (m < 0) m += period;
    return m < n ? m : period - 1 - m;
}

struct BruteArgs {
    const float* img;
    int width, height, r, R, border;
    const double* taps;   // 2r+1 (device)
    const double* range;  // 2R+1 (device)
    double* out;
    unsigned long long* fallbacks;
};

__global__ void __launch_bounds__(kBX* kBY) brute_kernel(const BruteArgs a) {
    extern __shared__ unsigned char smem_raw[];
    const int r = a.r, tw = kBX + 2 * r, th = kBY + 2 * r;
    const int nrange = 2 * a.R + 1;
    double* s_taps = reinterpret_cast<double*>(smem_raw);               // [2r+1]
    double* s_range = s_taps + (2 * r + 1);                              // [2R+1] if small
    float* tile = reinterpret_cast<float*>(s_range + (nrange <= kRangeSmem ? nrange : 0));  // [th][tw]
    const int tid = threadIdx.y * kBX + threadIdx.x;
    const int x0 = blockIdx.x * kBX, y0 = blockIdx.y * kBY;
    for (int i = tid; i < 2 * r + 1; i += kBX * kBY) s_taps[i] = a.taps[i];
    if (nrange <= kRangeSmem)
        for (int i = tid; i < nrange; i += kBX * kBY) s_range[i] = a.range[i];
    // input tile with the border mapping applied once; -1 marks a skipped sample
    // (zero border outside the image; intensities are validated to [0, R])
    for (int i = tid; i < tw * th; i += kBX * kBY) {
        const int ty = i / tw, tx = i - ty * tw;
        const int my = border_index(y0 - r + ty, a.height, a.border);
        const int mx = border_index(x0 - r + tx, a.width, a.border);
        tile[i] = (my < 0 || mx < 0) ? -1.0f : __ldg(a.img + (size_t)my * a.width + mx);
    }
    __syncthreads();
    const double* rng = nrange <= kRangeSmem ? s_range : a.range;
    const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
    unsigned fb = 0;
    if (x < a.width && y < a.height) {
        const double center = (double)tile[(threadIdx.y + r) * tw + threadIdx.x + r];
        double num = 0.0, den = 0.0;
        for (int dy = -r; dy <= r; ++dy) {
            const double wy = s_taps[r + dy];
            const float* row = tile + (threadIdx.y + r + dy) * tw + threadIdx.x + r;
            for (int dx = -r; dx <= r; ++dx) {
                const float v = row[dx];
                if (v < 0.0f) continue;
                const double nb = (double)v;
                const long long t = llround(__dsub_rn(nb, center));
                const double weight = __dmul_rn(__dmul_rn(wy, s_taps[r + dx]), rng[t + a.R]);
                num = __dadd_rn(num, __dmul_rn(weight, nb));
                den = __dadd_rn(den, weight);
            }
        }
        double o = center;
        if (den > 0.0) o = __ddiv_rn(num, den);
        else fb = 1;
        a.out[(size_t)y * a.width + x] = o;
    }
    if (a.fallbacks) {
        const unsigned w = __reduce_add_sync(0xffffffffu, fb);
        if ((threadIdx.x & 31) == 0 && w) atomicAdd(a.fallbacks, (unsigned long long)w);
    }
}

size_t brute_smem_bytes(int r, int R) {
    const int nrange = 2 * R + 1;
    return sizeof(double) * (2 * r + 1 + (nrange <= kRangeSmem ? nrange : 0)) +
           sizeof(float) * (size_t)(kBX + 2 * r) * (kBY + 2 * r);
}

// per-block (sum of squares, max |d|) of a (double) - b (float)
__global__ void __launch_bounds__(kCmpThreads) compare_kernel(const double* __restrict__ a, const float* __restrict__ b,
                                                              size_t n, double* __restrict__ part) {
    double s = 0.0, mx = 0.0;
    for (size_t i = (size_t)blockIdx.x * kCmpThreads + threadIdx.x; i < n; i += (size_t)gridDim.x * kCmpThreads) {
        const double d = a[i] - (double)b[i];
        s += d * d;
        mx = fmax(mx, fabs(d));
    }
    __shared__ double ss[kCmpThreads], sm[kCmpThreads];
    ss[threadIdx.x] = s;
    sm[threadIdx.x] = mx;
    __syncthreads();
    for (int o = kCmpThreads / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) {
            ss[threadIdx.x] += ss[threadIdx.x + o];
            sm[threadIdx.x] = fmax(sm[threadIdx.x], sm[threadIdx.x + o]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = ss[0];
        part[2 * blockIdx.x + 1] = sm[0];
    }
}

}  // namespace fbf_dev

namespace fbf_b200 {
namespace {

int cu_fail(cudaError_t e, const char* what) {
    return fail(FBF_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define FBF_CU(call, what)                                   \
    do {                                                     \
        cudaError_t e_ = (call);                             \
        if (e_ != cudaSuccess) return cu_fail(e_, what);     \
    } while (0)

int check_brute(int width, int height, double theta, const double* range, int R, int border, int* radius) {
    if (width < 1 || height < 1) return fail(FBF_EINVAL, "brute_bilateral: empty image");
    if (!(theta > 0.0) || !std::isfinite(theta))
        return fail(FBF_EINVAL, "spatial kernel: theta must be positive");  // kernels.cpp:106-107
    if (R < 1 || !range) return fail(FBF_EINVAL, "brute_bilateral: invalid range kernel samples");
    if (border < FBF_BORDER_SYMMETRIC || border > FBF_BORDER_ZERO)
        return fail(FBF_EINVAL, "brute_bilateral: unknown border policy");
    const int r = (int)std::ceil(3.0 * theta);
    if (r > fbf_dev::kBruteMaxRadius)
        return fail(FBF_ECAPACITY, "brute_bilateral: radius " + std::to_string(r) + " exceeds " +
                                       std::to_string(fbf_dev::kBruteMaxRadius));
    *radius = r;
    return FBF_OK;
}

// Launches the brute kernel on device buffers; `scratch` holds taps + range.
int launch_brute(const float* d_img, int width, int height, double theta, int r, const double* range, int R,
                 int border, double* d_out, unsigned long long* d_fallbacks, double* d_params, cudaStream_t st) {
    std::vector<double> params(2 * r + 1 + 2 * R + 1);
    if (fbf_build_spatial_kernel(theta, params.data(), 2 * r + 1) != r)
        return fail(FBF_EINVAL, "spatial kernel: theta must be positive");
    std::copy(range, range + 2 * R + 1, params.begin() + 2 * r + 1);
    FBF_CU(cudaMemcpyAsync(d_params, params.data(), sizeof(double) * params.size(), cudaMemcpyHostToDevice, st),
           "H2D params");
    fbf_dev::BruteArgs a{d_img, width, height, r, R, border, d_params, d_params + 2 * r + 1, d_out, d_fallbacks};
    const size_t smem = fbf_dev::brute_smem_bytes(r, R);
    FBF_CU(cudaFuncSetAttribute(fbf_dev::brute_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
           "smem attribute");
    dim3 grid((width + fbf_dev::kBX - 1) / fbf_dev::kBX, (height + fbf_dev::kBY - 1) / fbf_dev::kBY);
    fbf_dev::brute_kernel<<<grid, dim3(fbf_dev::kBX, fbf_dev::kBY), smem, st>>>(a);
    FBF_CU(cudaGetLastError(), "brute launch");
    count_launch();
    return FBF_OK;
}

struct DevBuf {
    void* p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    int alloc(size_t bytes) {
        if (cudaMalloc(&p, bytes) != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
            return fail(FBF_ENOMEM, "device allocation of " + std::to_string(bytes) + " bytes failed");
        }
        return FBF_OK;
    }
};

}  // namespace
}  // namespace fbf_b200

using namespace fbf_b200;

extern "C" {

int fbf_brute_bilateral_f32_device(const float* d_img, int width, int height, double theta, const double* range,
                                   int R, int border, double* d_out, unsigned long long* d_fallbacks, int device,
                                   void* stream) {
    int r = 0;
    int rc = check_brute(width, height, theta, range, R, border, &r);
    if (rc != FBF_OK) return rc;
    void* sv = nullptr;
    std::mutex* mtx = nullptr;
    if ((rc = device_context(device, &sv, &mtx)) != FBF_OK) return rc;
    DeviceGuard dguard;
    FBF_CU(cudaSetDevice(device), "cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    DevBuf params;
    if ((rc = params.alloc(sizeof(double) * (2 * r + 1 + 2 * R + 1))) != FBF_OK) return rc;
    rc = launch_brute(d_img, width, height, theta, r, range, R, border, d_out, d_fallbacks, (double*)params.p, st);
    if (rc != FBF_OK) return rc;
    FBF_CU(cudaStreamSynchronize(st), "brute");  // params are freed on return
    clear_error();
    return FBF_OK;
}

int fbf_brute_bilateral_f32(const float* img, int width, int height, double theta, const double* range, int R,
                            int border, double* out, long long* fallbacks) {
    int r = 0;
    int rc = check_brute(width, height, theta, range, R, border, &r);
    if (rc != FBF_OK) return rc;
    // validate_intensities (filter.cpp:19-23)
    const size_t n = (size_t)width * height;
    for (size_t i = 0; i < n; ++i)
        if (!(img[i] >= 0.0f && img[i] <= (float)R)) return fail(FBF_ERANGE, "filter: pixel intensity outside [0, R]");
    const int device = fbf_get_device();
    void* sv = nullptr;
    std::mutex* mtx = nullptr;
    if ((rc = device_context(device, &sv, &mtx)) != FBF_OK) return rc;
    std::lock_guard<std::mutex> lock(*mtx);
    DeviceGuard dguard;
    FBF_CU(cudaSetDevice(device), "cudaSetDevice");
    cudaStream_t st = (cudaStream_t)sv;
    DevBuf d_img, d_out, d_params, d_fb;
    if ((rc = d_img.alloc(sizeof(float) * n)) != FBF_OK) return rc;
    if ((rc = d_out.alloc(sizeof(double) * n)) != FBF_OK) return rc;
    if ((rc = d_params.alloc(sizeof(double) * (2 * r + 1 + 2 * R + 1))) != FBF_OK) return rc;
    if ((rc = d_fb.alloc(sizeof(unsigned long long))) != FBF_OK) return rc;
    FBF_CU(cudaMemcpyAsync(d_img.p, img, sizeof(float) * n, cudaMemcpyHostToDevice, st), "H2D");
    FBF_CU(cudaMemsetAsync(d_fb.p, 0, sizeof(unsigned long long), st), "memset");
    rc = launch_brute((const float*)d_img.p, width, height, theta, r, range, R, border, (double*)d_out.p,
                      (unsigned long long*)d_fb.p, (double*)d_params.p, st);
    if (rc != FBF_OK) return rc;
    unsigned long long nfb = 0;
    FBF_CU(cudaMemcpyAsync(out, d_out.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st), "D2H");
    FBF_CU(cudaMemcpyAsync(&nfb, d_fb.p, sizeof(nfb), cudaMemcpyDeviceToHost, st), "D2H");
    FBF_CU(cudaStreamSynchronize(st), "brute");
    if (fallbacks) *fallbacks += (long long)nfb;
    clear_error();
    return FBF_OK;
}

int fbf_compare_images_device(const double* d_ref, const float* d_cand, size_t n, double* mse, double* psnr_db,
                              double* max_abs, int device, void* stream) {
    if (n == 0) return fail(FBF_EINVAL, "compare_images: empty images");
    int rc = FBF_OK;
    void* sv = nullptr;
    std::mutex* mtx = nullptr;
    if ((rc = device_context(device, &sv, &mtx)) != FBF_OK) return rc;
    DeviceGuard dguard;
    FBF_CU(cudaSetDevice(device), "cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    DevBuf part;
    if ((rc = part.alloc(sizeof(double) * 2 * fbf_dev::kCmpBlocks)) != FBF_OK) return rc;
    fbf_dev::compare_kernel<<<fbf_dev::kCmpBlocks, fbf_dev::kCmpThreads, 0, st>>>(d_ref, d_cand, n, (double*)part.p);
    FBF_CU(cudaGetLastError(), "compare launch");
    count_launch();
    std::vector<double> h(2 * fbf_dev::kCmpBlocks);
    FBF_CU(cudaMemcpyAsync(h.data(), part.p, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, st), "D2H");
    FBF_CU(cudaStreamSynchronize(st), "compare");
    double s = 0.0, mx = 0.0;
    for (int b = 0; b < fbf_dev::kCmpBlocks; ++b) {
        s += h[2 * b];
        mx = std::max(mx, h[2 * b + 1]);
    }
    const double m = s / (double)n;
    if (mse) *mse = m;
    if (max_abs) *max_abs = mx;
    // metrics.cpp:22-23
    if (psnr_db) *psnr_db = m > 0.0 ? 10.0 * std::log10(255.0 * 255.0 / m) : INFINITY;
    clear_error();
    return FBF_OK;
}

}  // extern "C"
