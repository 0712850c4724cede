// fbf_kernel.cuh -- the fused Fourier bilateral filtering kernel for sm_100a.
//
// Replaces, in ONE launch per coefficient chunk, the reference's
//   fast_bilateral aux-image generation   (src/filter.cpp:164-177)
//   4K-2 x convolve_separable             (src/filter.cpp:74-81, 152-154, 182-185)
//     = convolve_rows (:27-49) + convolve_cols (:52-70) + map_border_index
//       (include/fourierbf/image.hpp:43-61)
//   per-term accumulation                 (src/filter.cpp:157-160, 189-194)
//   combine + fallback                    (src/filter.cpp:197-211)
// without materialising any of the 4K-2 auxiliary images in HBM.
//
// Dataflow (one persistent CTA per SM, column strips streamed top to bottom):
//   * The image is cut into strips of TW=32 output columns. Each CTA owns a
//     contiguous range of (frame, strip, row) units, i.e. one or a few strip
//     segments, so every SM gets the same number of output rows.
//   * A segment is streamed in steps of Q=16 input rows. Per step:
//       gen  : f for the Q new rows x (TW + 2r) columns (border-mapped), and
//              the channel pairs (f, 1) for k = 0 and (C_k f, S_k f), (C_k, S_k)
//              for k >= 1, C_k + i S_k = exp(i k nu f), into shared memory.
//       row  : horizontal (2r+1)-tap pass of every channel pair, P=8 outputs
//              per thread, packed FFMA2 with the tap broadcast from a uniform
//              register; results go to a ring of Q + 2r rows.
//       col  : vertical pass over the ring, P=8 outputs per thread, FFMA2.
//       comb : per output pixel, num += c_k (C_k G(C_k f) + S_k G(S_k f)),
//              den += c_k (C_k G(C_k) + S_k G(S_k)) in ascending k, then
//              out = den > 1e-12 ? num / den : f.
//   * Channel pairs share taps, so one FFMA2 advances two channels (the
//     reference's 4K-2 channels are exactly 2K-1 pairs).
//   * Coefficient chunks: when 2K-1 pairs do not fit in shared memory the
//     host launches one pass per chunk of k; (num, den) are carried in a
//     float2 scratch image between passes, still in ascending k.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fbf_dev {

constexpr int kTW = 32;          // output columns per strip
constexpr int kQ = 16;           // input rows per pipeline step
constexpr int kP = 8;            // outputs per thread item (row and column passes)
constexpr int kMaxPairs = 10;    // channel pairs per launch (block = 64 * pairs threads)
constexpr int kMaxKC = kMaxPairs / 2 + 1;  // k values per launch
constexpr int kMaxRadius = 32;
constexpr int kItemsPerPair = kQ * kTW / kP;  // 64 threads per channel pair
constexpr size_t kSmemLimit = 232448;          // 227 KB opt-in per block on sm_100

struct Params {
    const float* src;            // frame 0, global row src_row0, column 0
    long long src_frame_stride;  // floats between frames
    int src_pitch;               // floats between rows
    int src_row0, src_rows;      // global rows present in src
    float* dst;                  // frame 0, global row out_row0
    long long dst_frame_stride;
    int dst_pitch;
    float2* acc;                 // (num, den) scratch for multi-chunk runs, pitch = width
    long long acc_frame_stride;
    unsigned long long* fallbacks;  // device counter (may be null)
    int width, height, n_frames, border;
    int out_row0, out_rows;
    int k_lo, n_k, n_pairs;
    int first_chunk, last_chunk;
    int n_strips;
    long long total_units;  // n_frames * n_strips * out_rows
    float taps[kMaxRadius + 1];  // taps[j] = exp(-j^2 / (2 theta^2)), j = |d|
    float coeff[kMaxKC];
    double kinv[kMaxKC];         // k / (2T + 1) for the chunk's k values
};

template <int R>
struct Geometry {
    static constexpr int GW = kTW + 2 * R;                       // gen row width (pixels)
    static constexpr int GS = GW + ((2 - GW % 4) + 4) % 4;       // stride, GS/2 odd
    static constexpr int RING = kQ + 2 * R;                      // ring rows
    static constexpr int RS = kTW + 2;                           // ring stride, RS/2 odd
    static constexpr size_t pair_bytes = sizeof(float2) * (size_t)(kQ * GS + RING * RS);
    static constexpr size_t fixed_bytes = sizeof(float) * (size_t)(RING * kTW) + 16;
    static size_t smem_bytes(int pairs) { return fixed_bytes + pair_bytes * pairs; }
    static int max_pairs() {
        const size_t p = (kSmemLimit - fixed_bytes) / pair_bytes;
        return (int)(p < (size_t)kMaxPairs ? p : (size_t)kMaxPairs);
    }
};

// image.hpp:43-61
__host__ __device__ __forceinline__ int map_border(int i, int n, int border) {
    if (i >= 0 && i < n) return i;
    if (border == 2) return -1;
    if (border == 1) return i < 0 ? 0 : n - 1;
    const int period = 2 * n;
    int m = i % period;
    if (m < 0) m += period;
    return m < n ? m : period - 1 - m;
}

// (cos, sin)(2 pi * k f / (2T+1)): exact turn reduction in double, then the
// MUFU pair on [-pi, pi]. Used identically by gen and combine, so the
// modulation and demodulation factors agree bit for bit.
__device__ __forceinline__ float2 harmonic(float f, double kinv) {
    double t = (double)f * kinv;
    t -= rint(t);
    const float th = (float)(t * 6.283185307179586476925286766559);
    float s, c;
    __sincosf(th, &s, &c);
    return make_float2(c, s);
}

__device__ __forceinline__ float2 ffma2(float2 a, float w, float2 c) {
    return __ffma2_rn(a, make_float2(w, w), c);
}

template <int R>
__global__ void __launch_bounds__(kMaxPairs * kItemsPerPair, 1) fbf_fused_kernel(const Params p) {
    using G = Geometry<R>;
    constexpr int GW = G::GW, GS = G::GS, RING = G::RING, RS = G::RS;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int np = p.n_pairs;
    float2* gen = reinterpret_cast<float2*>(smem_raw);       // [np][Q][GS]; later colout [np][Q][TW]
    float2* ring = gen + (size_t)np * kQ * GS;                // [np][RING][RS]
    float* fring = reinterpret_cast<float*>(ring + (size_t)np * RING * RS);  // [RING][TW]
    unsigned int* s_fallbacks = reinterpret_cast<unsigned int*>(fring + RING * kTW);
    float2* colout = gen;

    const int tid = threadIdx.x;
    const int nthreads = blockDim.x;
    if (tid == 0) *s_fallbacks = 0u;

    // this CTA's contiguous share of the (frame, strip, row) units
    const long long U = p.total_units;
    const long long u_begin = U * blockIdx.x / gridDim.x;
    const long long u_end = U * (blockIdx.x + 1) / gridDim.x;
    const long long per_frame = (long long)p.n_strips * p.out_rows;

    for (long long u = u_begin; u < u_end;) {
        const int frame = (int)(u / per_frame);
        const long long rem = u % per_frame;
        const int strip = (int)(rem / p.out_rows);
        const int row = (int)(rem % p.out_rows);
        const int len = (int)min((long long)(p.out_rows - row), u_end - u);
        u += len;

        const int x0 = strip * kTW;
        const int ya = p.out_row0 + row, yb = ya + len;
        const float* src = p.src + (long long)frame * p.src_frame_stride;
        float* dst = p.dst + (long long)frame * p.dst_frame_stride;
        float2* acc = p.acc ? p.acc + (long long)frame * p.acc_frame_stride : nullptr;

        // steps start e rows early so that output rows begin exactly at ya
        constexpr int e = (kQ - (2 * R) % kQ) % kQ;
        constexpr int s0 = (2 * R + e) / kQ;
        const int a0 = ya - R - e;
        const int steps = s0 + (len + kQ - 1) / kQ;

        for (int s = 0; s < steps; ++s) {
            const int a = a0 + s * kQ;
            const int slot_base = (s * kQ) % RING;
            __syncthreads();  // previous step's combine is done with colout/fring

            // ---- gen: channel pairs of the Q new input rows -------------------
            for (int pix = tid; pix < kQ * GW; pix += nthreads) {
                const int q = pix / GW, xl = pix - q * GW;
                const int gy = a + q, gx = x0 - R + xl;
                const bool need = gy >= ya - R && gy < yb + R;
                const int my = need ? map_border(gy, p.height, p.border) : -1;
                const int mx = map_border(gx, p.width, p.border);
                const bool valid = my >= 0 && mx >= 0;
                const float f = valid ? __ldg(src + (long long)(my - p.src_row0) * p.src_pitch + mx) : 0.f;
                if (xl >= R && xl < R + kTW) fring[((slot_base + q) % RING) * kTW + (xl - R)] = f;
                float2* g = gen + q * GS + xl;
                int pi = 0;
                for (int kk = 0; kk < p.n_k; ++kk) {
                    if (p.k_lo + kk == 0) {
                        g[(size_t)pi * kQ * GS] = valid ? make_float2(f, 1.f) : make_float2(0.f, 0.f);
                        pi += 1;
                    } else {
                        float2 cs = harmonic(f, p.kinv[kk]);
                        if (!valid) cs = make_float2(0.f, 0.f);
                        g[(size_t)pi * kQ * GS] = make_float2(cs.x * f, cs.y * f);
                        g[(size_t)(pi + 1) * kQ * GS] = cs;
                        pi += 2;
                    }
                }
            }
            __syncthreads();

            // ---- row pass: horizontal taps, ring[pair][slot][x] ----------------
            {  // blockDim.x == n_items: one item per thread
                const int q = tid % kQ;
                const int xc = (tid / kQ) % (kTW / kP);
                const int pr = tid / (kQ * (kTW / kP));
                const float4* gin = reinterpret_cast<const float4*>(gen + ((size_t)pr * kQ + q) * GS + xc * kP);
                float2 accp[kP];
#pragma unroll
                for (int o = 0; o < kP; ++o) accp[o] = make_float2(0.f, 0.f);
#pragma unroll
                for (int j = 0; j < (kP + 2 * R) / 2; ++j) {
                    const float4 v4 = gin[j];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int jj = 2 * j + h;
                        const float2 v = h ? make_float2(v4.z, v4.w) : make_float2(v4.x, v4.y);
#pragma unroll
                        for (int o = 0; o < kP; ++o) {
                            const int d = jj - o;  // tap index 0..2R, ascending per output
                            if (d >= 0 && d <= 2 * R) accp[o] = ffma2(v, p.taps[d >= R ? d - R : R - d], accp[o]);
                        }
                    }
                }
                float4* hout = reinterpret_cast<float4*>(ring + ((size_t)pr * RING + (slot_base + q) % RING) * RS + xc * kP);
#pragma unroll
                for (int o = 0; o < kP / 2; ++o)
                    hout[o] = make_float4(accp[2 * o].x, accp[2 * o].y, accp[2 * o + 1].x, accp[2 * o + 1].y);
            }
            __syncthreads();
            if (s < s0) continue;  // warm-up: the ring is not full yet

            // ---- column pass: vertical taps over the ring -> colout ------------
            // (gen was last read by the row pass, so colout may overwrite it)
            {
                const int x = tid % kTW;
                const int g = (tid / kTW) % (kQ / kP);
                const int pr = tid / (kTW * (kQ / kP));
                const int q0 = g * kP;
                const float2* rp = ring + (size_t)pr * RING * RS + x;
                int sl = (slot_base + kQ + q0) % RING;
                float2 accp[kP];
#pragma unroll
                for (int o = 0; o < kP; ++o) accp[o] = make_float2(0.f, 0.f);
#pragma unroll
                for (int i = 0; i < kP + 2 * R; ++i) {
                    const float2 v = rp[sl * RS];
                    sl = (sl + 1 == RING) ? 0 : sl + 1;
#pragma unroll
                    for (int o = 0; o < kP; ++o) {
                        const int d = i - o;
                        if (d >= 0 && d <= 2 * R) accp[o] = ffma2(v, p.taps[d >= R ? d - R : R - d], accp[o]);
                    }
                }
#pragma unroll
                for (int o = 0; o < kP; ++o) colout[((size_t)pr * kQ + q0 + o) * kTW + x] = accp[o];
            }
            __syncthreads();

            // ---- combine ------------------------------------------------------
            for (int pix = tid; pix < kQ * kTW; pix += nthreads) {
                const int q = pix / kTW, x = pix - q * kTW;
                const int y = a - R + q, gxo = x0 + x;
                if (y >= yb || gxo >= p.width) continue;
                const float f = fring[((slot_base + kQ + R + q) % RING) * kTW + x];
                float num = 0.f, den = 0.f;
                const long long ai = (long long)(y - p.out_row0) * p.width + gxo;
                if (!p.first_chunk) {
                    const float2 nd = acc[ai];
                    num = nd.x;
                    den = nd.y;
                }
                int pi = 0;
                for (int kk = 0; kk < p.n_k; ++kk) {
                    const float ck = p.coeff[kk];
                    if (p.k_lo + kk == 0) {
                        const float2 g0 = colout[((size_t)pi * kQ + q) * kTW + x];
                        num += ck * g0.x;
                        den += ck * g0.y;
                        pi += 1;
                    } else {
                        const float2 cs = harmonic(f, p.kinv[kk]);
                        const float2 gn = colout[((size_t)pi * kQ + q) * kTW + x];
                        const float2 gd = colout[((size_t)(pi + 1) * kQ + q) * kTW + x];
                        num += ck * (cs.x * gn.x + cs.y * gn.y);
                        den += ck * (cs.x * gd.x + cs.y * gd.y);
                        pi += 2;
                    }
                }
                if (p.last_chunk) {
                    float o = f;
                    if (den > 1e-12f) o = num / den;
                    else atomicAdd(s_fallbacks, 1u);
                    dst[(long long)(y - p.out_row0) * p.dst_pitch + gxo] = o;
                } else {
                    acc[ai] = make_float2(num, den);
                }
            }
        }
    }
    __syncthreads();
    if (tid == 0 && p.fallbacks && *s_fallbacks) atomicAdd(p.fallbacks, (unsigned long long)*s_fallbacks);
}

template <int R>
cudaError_t launch_fused(const Params& p, int grid, cudaStream_t stream) {
    using G = Geometry<R>;
    const size_t smem = G::smem_bytes(p.n_pairs);
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(fbf_fused_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)kSmemLimit);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    fbf_fused_kernel<R><<<grid, p.n_pairs * kItemsPerPair, smem, stream>>>(p);
    return cudaGetLastError();
}

}  // namespace fbf_dev
