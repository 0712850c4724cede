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
// Dataflow (persistent CTAs, column strips streamed top to bottom, two
// warp-specialised roles connected by mbarriers so that the latency-bound
// phases of one overlap the FFMA2-bound phases of the other):
//   * The image is cut into strips of TW=32 output columns. Each CTA owns a
//     contiguous range of (frame, strip, row) units -- one or a few strip
//     segments -- so every CTA gets the same number of output rows.
//   * A segment is streamed in steps of Q=8 input rows. Producer warps run
//     stage + gen + row for step s while consumer warps run col + comb for
//     step s-1; ring blocks are handed over with full/empty mbarriers.
//       stage: the f tile of the NEXT step (Q rows x (TW+2r) columns) is
//              fetched asynchronously: one TMA bulk copy per row
//              (cp.async.bulk, mbarrier complete_tx) for interior tiles,
//              border-mapped per-pixel cp.async at the image edges (the copy
//              engine cannot mirror).
//       gen  : channel pairs (f, 1) for k = 0 and (C_k f, S_k f), (C_k, S_k)
//              for k >= 1, with C_k + i S_k = exp(i k nu f) from one
//              double-reduced MUFU sincos and the angle-addition recurrence.
//       row  : horizontal (2r+1)-tap pass of every channel pair, 8 outputs
//              per thread, FFMA2 with the tap broadcast from a uniform
//              register; results go to a ring of 1 + ceil(2r/Q) row blocks.
//       col  : vertical pass over the ring, 8 outputs per thread, FFMA2; the
//              ring window resolves to fixed offsets at compile time.
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
constexpr int kQ = 8;            // input rows per pipeline step
constexpr int kP = 8;            // outputs per thread item (row and column passes)
constexpr int kMaxKR = 7;        // k >= 1 terms per launch (template parameter NKR <= kMaxKR)
constexpr int kMaxPairs = 1 + 2 * kMaxKR;
constexpr int kMaxRadius = 32;
constexpr int kItemsPerPair = kQ * kTW / kP;  // 32 threads (one warp) per channel pair and role
constexpr int kMaxThreads = 2 * kMaxPairs * kItemsPerPair;
constexpr size_t kSmemLimit = 232448;          // 227 KB opt-in per block on sm_100
constexpr size_t kSmemPerSM = 233472;          // 228 KB per SM
constexpr size_t kSmemReservedPerBlock = 1024;

static_assert(kQ == kP, "one column-pass row group per step");

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
    int k_lo, n_pairs;           // chunk: k in [k_lo, k_lo + (k_lo == 0) + NKR)
    int k_first;                 // first k >= 1 of the chunk
    int first_chunk, last_chunk;
    int n_strips;
    int use_tma;
    long long total_units;       // n_frames * n_strips * out_rows
    float taps[kMaxRadius + 1];  // taps[j] = exp(-j^2 / (2 theta^2)), j = |d|
    float coeff[kMaxKR + 1];     // c_k of the chunk, ascending k
    float inv_period;            // 1 / (2T + 1)
};

template <int R>
struct Geometry {
    static constexpr int GW = kTW + 2 * R;                       // gen row width (pixels)
    static constexpr int GS = GW + ((2 - GW % 4) + 4) % 4;       // gen stride (float2), GS/2 odd
    static constexpr int FSW = (GW + 3 + 3) / 4 * 4;             // f staging row: GW + 16B-alignment slack
    static constexpr int RB = 1 + (2 * R + kQ - 1) / kQ;         // ring blocks a column pass reads
    static constexpr int RBX = RB + 1;                           // + the block being produced
    static constexpr int RROWS = RBX * kQ;                       // ring rows
    static constexpr int RS = kTW + 2;                           // ring stride (float2), RS/2 odd
    static constexpr size_t fstage_bytes = sizeof(float) * 2 * kQ * FSW;  // multiple of 128
    static constexpr size_t bar_bytes = 8 * (2 + 2 * RBX) + 8;            // mbarriers + counter
    static constexpr size_t misc_bytes = (bar_bytes + 127) / 128 * 128;
    static constexpr size_t colmap_bytes = sizeof(int) * ((GW + 3) / 4 * 4);
    static constexpr size_t fring_bytes = sizeof(float) * RROWS * kTW;
    static constexpr size_t fixed_bytes = fstage_bytes + misc_bytes + colmap_bytes + fring_bytes;
    static constexpr size_t pair_bytes = sizeof(float2) * (size_t)(kQ * GS + kQ * kTW + RROWS * RS);
    static size_t smem_bytes(int pairs) { return fixed_bytes + pair_bytes * pairs; }
    static int max_pairs(int blocks_per_sm) {
        size_t budget = kSmemPerSM / blocks_per_sm - kSmemReservedPerBlock;
        if (budget > kSmemLimit) budget = kSmemLimit;
        if (budget <= fixed_bytes) return 0;
        const size_t p = (budget - fixed_bytes) / pair_bytes;
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

// (cos, sin)(2 pi f / (2T+1)): turn reduction (exact: |t| < 1), then the MUFU
// pair on [-pi, pi].
__device__ __forceinline__ float2 harmonic1(float f, float inv_period) {
    float t = f * inv_period;
    t -= rintf(t);
    float s, c;
    __sincosf(t * 6.28318530717958647692f, &s, &c);
    return make_float2(c, s);
}

// exp(i (k+1) w) = exp(i k w) * exp(i w). gen and combine run this identical
// sequence, so modulation and demodulation factors agree bit for bit and do not
// depend on how k is split into chunks.
__device__ __forceinline__ float2 rotate(float2 cs, float2 c1) {
    return make_float2(fmaf(cs.x, c1.x, -(cs.y * c1.y)), fmaf(cs.y, c1.x, cs.x * c1.y));
}

__device__ __forceinline__ float2 harmonic_first(float2 c1, int k_first) {
    float2 cs = c1;
    for (int k = 1; k < k_first; ++k) cs = rotate(cs, c1);
    return cs;
}

__device__ __forceinline__ float2 ffma2(float2 a, float w, float2 c) {
    return __ffma2_rn(a, make_float2(w, w), c);
}

// ---- synchronisation / async copy primitives -------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void named_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void cp_async4(float* smem_dst, const float* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(smem_dst)), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
// 1-D TMA bulk copy global -> shared (16-byte aligned, size multiple of 16),
// completion on `bar`.
__device__ __forceinline__ void tma_bulk_g2s(float* smem_dst, const float* gsrc, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(smem_dst)),
                 "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// Vertical pass for the kQ output rows of global step g. The window rows
// j in [-2R, kP) (relative to block g) resolve to (block, row) at compile
// time, so every load is a fixed offset from one of RB block pointers.
template <int R>
__device__ __forceinline__ void column_pass(const float2* __restrict__ ring_pair, int blk, int x,
                                            const float* taps, float2* out_col) {
    using G = Geometry<R>;
    constexpr int RB = G::RB, RBX = G::RBX, RS = G::RS;
    const float2* bptr[RB];
#pragma unroll
    for (int b = 0; b < RB; ++b) {  // bptr[b] = block (blk - b) mod RBX
        int bb = blk - b;
        bb += bb < 0 ? RBX : 0;
        bptr[b] = ring_pair + bb * kQ * RS + x;
    }
    float2 acc[kP];
#pragma unroll
    for (int o = 0; o < kP; ++o) acc[o] = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < kP + 2 * R; ++i) {
        const int j = i - 2 * R;                          // compile-time
        const int b = j >= 0 ? 0 : (-j + kQ - 1) / kQ;    // blocks back
        const float2 v = bptr[b][(j + b * kQ) * RS];
#pragma unroll
        for (int o = 0; o < kP; ++o) {
            const int d = i - o;
            if (d >= 0 && d <= 2 * R) acc[o] = ffma2(v, taps[d >= R ? d - R : R - d], acc[o]);
        }
    }
#pragma unroll
    for (int o = 0; o < kP; ++o) out_col[o * kTW] = acc[o];
}

template <int R, int NKR>
__global__ void __launch_bounds__(2 * (1 + 2 * NKR) * kItemsPerPair, 1) fbf_fused_kernel(const __grid_constant__ Params p) {
    using G = Geometry<R>;
    constexpr int GW = G::GW, GS = G::GS, FSW = G::FSW, RB = G::RB, RBX = G::RBX, RROWS = G::RROWS, RS = G::RS;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int np = p.n_pairs;
    float* fstage = reinterpret_cast<float*>(smem_raw);                         // [2][Q][FSW]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + G::fstage_bytes);   // fs[2], full[RBX], empty[RBX]
    uint64_t* fs_bar = bars;
    uint64_t* full_bar = bars + 2;
    uint64_t* empty_bar = bars + 2 + RBX;
    unsigned int* s_fallbacks = reinterpret_cast<unsigned int*>(bars + 2 + 2 * RBX);
    int* colmap = reinterpret_cast<int*>(smem_raw + G::fstage_bytes + G::misc_bytes);  // [GW]
    float* fring = reinterpret_cast<float*>(smem_raw + G::fstage_bytes + G::misc_bytes + G::colmap_bytes);
    float2* gen = reinterpret_cast<float2*>(fring + RROWS * kTW);  // [np][Q][GS]     (producer)
    float2* colout = gen + (size_t)np * kQ * GS;                   // [np][Q][TW]     (consumer)
    float2* ring = colout + (size_t)np * kQ * kTW;                 // [np][RROWS][RS] (handoff)

    const int nrole = np * kItemsPerPair;  // threads per role
    const bool producer = threadIdx.x < nrole;
    const int tid = producer ? threadIdx.x : threadIdx.x - nrole;
    const int zk = p.k_lo == 0 ? 1 : 0;  // k = 0 contributes the single pair (f, 1)
    if (threadIdx.x == 0) {
        *s_fallbacks = 0u;
        mbar_init(&fs_bar[0], 1);
        mbar_init(&fs_bar[1], 1);
        for (int b = 0; b < RBX; ++b) {
            mbar_init(&full_bar[b], 1);
            mbar_init(&empty_bar[b], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    unsigned fs_phase0 = 0, fs_phase1 = 0;

    // this CTA's contiguous share of the (frame, strip, row) units
    const long long U = p.total_units;
    const long long u_begin = U * blockIdx.x / gridDim.x;
    const long long u_end = U * (blockIdx.x + 1) / gridDim.x;
    const long long per_frame = (long long)p.n_strips * p.out_rows;
    int gstep = 0;  // global step counter: ring block = step % RBX

    for (long long u = u_begin; u < u_end;) {
        const int frame = (int)(u / per_frame);
        const long long rem = u % per_frame;
        const int strip = (int)(rem / p.out_rows);
        const int row = (int)(rem % p.out_rows);
        const int len = (int)min((long long)(p.out_rows - row), u_end - u);
        u += len;

        const int x0 = strip * kTW;
        const int ya = p.out_row0 + row, yb = ya + len;
        // steps start e rows early so that output rows begin exactly at ya
        constexpr int e = (kQ - (2 * R) % kQ) % kQ;
        constexpr int s0 = (2 * R + e) / kQ;
        const int a0 = ya - R - e;
        const int steps = s0 + (len + kQ - 1) / kQ;

        if (producer) {
            // =========================== PRODUCER ===========================
            const float* src = p.src + (long long)frame * p.src_frame_stride;
            // interior strips copy 16-byte-aligned row spans [xs, xs + FSW) with the copy engine
            const int xs = (x0 - R) & ~3, xoff = (x0 - R) - xs;
            const bool cols_interior = p.use_tma && xs >= 0 && xs + FSW <= p.width;
            named_sync(1, nrole);  // previous segment done with fstage / colmap
            for (int xl = tid; xl < GW; xl += nrole) colmap[xl] = map_border(x0 - R + xl, p.width, p.border);
            named_sync(1, nrole);

            // Stage the f tile of step `st` into fstage[st & 1]; returns whether TMA was used.
            auto stage_f = [&](int st) -> bool {
                float* fs = fstage + (st & 1) * kQ * FSW;
                const int a = a0 + st * kQ;
                const int lo = max(a, ya - R), hi = min(a + kQ, yb + R);
                if (cols_interior && lo >= 0 && hi <= p.height && lo < hi) {
                    if (tid < 32) {  // warp 0: one bulk copy per needed row
                        if (tid == 0) {
                            fence_proxy_async();
                            mbar_arrive_expect_tx(&fs_bar[st & 1], (unsigned)(sizeof(float) * FSW * (hi - lo)));
                        }
                        __syncwarp();
                        const int gy = lo + tid;
                        if (gy < hi)
                            tma_bulk_g2s(fs + (gy - a) * FSW, src + (long long)(gy - p.src_row0) * p.src_pitch + xs,
                                         (unsigned)(sizeof(float) * FSW), &fs_bar[st & 1]);
                    }
                    return true;
                }
                for (int pix = tid; pix < kQ * GW; pix += nrole) {
                    const int q = pix / GW, xl = pix - q * GW;
                    const int gy = a + q;
                    const int my = (gy >= lo && gy < hi) ? map_border(gy, p.height, p.border) : -1;
                    const int mx = colmap[xl];
                    float* d = fs + q * FSW + xoff + xl;
                    if (my >= 0 && mx >= 0)
                        cp_async4(d, src + (long long)(my - p.src_row0) * p.src_pitch + mx);
                    else
                        *d = 0.f;
                }
                cp_async_commit();
                return false;
            };
            bool tma_next = stage_f(0);

            for (int s = 0; s < steps; ++s) {
                const int g = gstep + s;
                const int blk = g % RBX;
                const int a = a0 + s * kQ;
                if (tma_next) {
                    if (s & 1) { mbar_wait(&fs_bar[1], fs_phase1); fs_phase1 ^= 1u; }
                    else       { mbar_wait(&fs_bar[0], fs_phase0); fs_phase0 ^= 1u; }
                }
                cp_async_wait_all();
                named_sync(1, nrole);  // fstage[s&1] complete; gen buffer free (row pass s-1 done)
                tma_next = (s + 1 < steps) ? stage_f(s + 1) : false;
                // ring/fring block `blk` is free once the consumer finished step g - 2
                if (g >= RBX) mbar_wait(&empty_bar[blk], (unsigned)((g / RBX - 1) & 1));

                // ---- gen: channel pairs of the Q new input rows ----------------
                {
                    const float* fs = fstage + (s & 1) * kQ * FSW;
                    const int lo = max(a, ya - R), hi = min(a + kQ, yb + R);
                    for (int pix = tid; pix < kQ * GW; pix += nrole) {
                        const int q = pix / GW, xl = pix - q * GW;
                        const int gy = a + q;
                        const bool valid = gy >= lo && gy < hi && colmap[xl] >= 0 &&
                                           (p.border != 2 || (gy >= 0 && gy < p.height));
                        const float f = valid ? fs[q * FSW + xoff + xl] : 0.f;
                        if (xl >= R && xl < R + kTW) fring[(blk * kQ + q) * kTW + (xl - R)] = f;
                        float2* gp = gen + q * GS + xl;
                        if (zk) gp[0] = valid ? make_float2(f, 1.f) : make_float2(0.f, 0.f);
                        if (NKR > 0) {
                            const float2 c1 = harmonic1(f, p.inv_period);
                            float2 cs = harmonic_first(c1, p.k_first);
                            if (!valid) cs = make_float2(0.f, 0.f);
                            float2* gk = gp + (size_t)zk * kQ * GS;
#pragma unroll
                            for (int kk = 0; kk < NKR; ++kk) {
                                gk[(size_t)(2 * kk) * kQ * GS] = make_float2(cs.x * f, cs.y * f);
                                gk[(size_t)(2 * kk + 1) * kQ * GS] = cs;
                                if (kk + 1 < NKR) cs = rotate(cs, c1);
                            }
                        }
                    }
                }
                named_sync(1, nrole);

                // ---- row pass: horizontal taps into ring block blk -------------
                {  // nrole == np * kItemsPerPair: one item per producer thread
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
                                if (d >= 0 && d <= 2 * R)
                                    accp[o] = ffma2(v, p.taps[d >= R ? d - R : R - d], accp[o]);
                            }
                        }
                    }
                    float4* hout =
                        reinterpret_cast<float4*>(ring + ((size_t)pr * RROWS + blk * kQ + q) * RS + xc * kP);
#pragma unroll
                    for (int o = 0; o < kP / 2; ++o)
                        hout[o] = make_float4(accp[2 * o].x, accp[2 * o].y, accp[2 * o + 1].x, accp[2 * o + 1].y);
                }
                named_sync(1, nrole);                   // every row of block blk written
                if (tid == 0) mbar_arrive(&full_bar[blk]);  // release to the consumer
            }
        } else {
            // =========================== CONSUMER ===========================
            float* dst = p.dst + (long long)frame * p.dst_frame_stride;
            float2* acc = p.acc ? p.acc + (long long)frame * p.acc_frame_stride : nullptr;
            for (int s = 0; s < steps; ++s) {
                const int g = gstep + s;
                const int blk = g % RBX;
                const int a = a0 + s * kQ;
                mbar_wait(&full_bar[blk], (unsigned)((g / RBX) & 1));
                if (s >= s0) {  // warm-up steps only fill the ring
                    // ---- column pass: vertical taps over the ring -> colout ----
                    {
                        const int x = tid % kTW;
                        const int pr = tid / kTW;
                        column_pass<R>(ring + (size_t)pr * RROWS * RS, blk, x, p.taps,
                                       colout + (size_t)pr * kQ * kTW + x);
                    }
                    named_sync(2, nrole);

                    // ---- combine -----------------------------------------------
                    for (int pix = tid; pix < kQ * kTW; pix += nrole) {
                        const int q = pix / kTW, x = pix - q * kTW;
                        const int y = a - R + q, gxo = x0 + x;
                        if (y >= yb || gxo >= p.width) continue;
                        int fr = blk * kQ + q - R;
                        while (fr < 0) fr += RROWS;
                        const float f = fring[fr * kTW + x];
                        float num = 0.f, den = 0.f;
                        const long long ai = (long long)(y - p.out_row0) * p.width + gxo;
                        if (!p.first_chunk) {
                            const float2 nd = acc[ai];
                            num = nd.x;
                            den = nd.y;
                        }
                        const float2* go = colout + q * kTW + x;
                        if (zk) {
                            const float2 g0 = go[0];
                            num += p.coeff[0] * g0.x;
                            den += p.coeff[0] * g0.y;
                        }
                        if (NKR > 0) {
                            const float2 c1 = harmonic1(f, p.inv_period);
                            float2 cs = harmonic_first(c1, p.k_first);
                            const float2* gk = go + (size_t)zk * kQ * kTW;
#pragma unroll
                            for (int kk = 0; kk < NKR; ++kk) {
                                const float ck = p.coeff[zk + kk];
                                const float2 gn = gk[(size_t)(2 * kk) * kQ * kTW];
                                const float2 gd = gk[(size_t)(2 * kk + 1) * kQ * kTW];
                                num += ck * (cs.x * gn.x + cs.y * gn.y);
                                den += ck * (cs.x * gd.x + cs.y * gd.y);
                                if (kk + 1 < NKR) cs = rotate(cs, c1);
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
                named_sync(2, nrole);  // all consumer reads of the ring / colout done
                // the oldest block of this step's window is no longer needed
                if (tid == 0 && g - RB + 1 >= 0) mbar_arrive(&empty_bar[(g - RB + 1) % RBX]);
            }
        }
        gstep += steps;
    }
    __syncthreads();
    if (threadIdx.x == 0 && p.fallbacks && *s_fallbacks) atomicAdd(p.fallbacks, (unsigned long long)*s_fallbacks);
}

template <int R, int NKR>
cudaError_t launch_fused(const Params& p, int grid, cudaStream_t stream) {
    using G = Geometry<R>;
    const size_t smem = G::smem_bytes(p.n_pairs);
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(fbf_fused_kernel<R, NKR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)kSmemLimit);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    fbf_fused_kernel<R, NKR><<<grid, 2 * p.n_pairs * kItemsPerPair, smem, stream>>>(p);
    return cudaGetLastError();
}

}  // namespace fbf_dev
