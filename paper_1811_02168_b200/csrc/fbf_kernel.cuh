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
//       stage: a loader warp fetches f tiles (Q rows x (TW+2r) columns) up to
//              three steps ahead: one TMA bulk copy per row (cp.async.bulk,
//              mbarrier complete_tx) for interior tiles, border-mapped
//              element loads at the image edges (the copy engine cannot mirror).
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
#ifndef FBF_Q
#define FBF_Q 8
#endif
constexpr int kQ = FBF_Q;        // input rows per pipeline step
constexpr int kP = 8;            // outputs per thread item (row and column passes)
constexpr int kMaxKR = 4;        // k >= 1 terms per launch (template parameter NKR <= kMaxKR)
constexpr int kMaxPairs = 1 + 2 * kMaxKR;
constexpr int kMaxRadius = 32;
constexpr int kItemsPerPair = kQ * kTW / kP;  // 32 threads (one warp) per channel pair and role
constexpr int kRoles = 2;        // pair warps and gen warps scale with the pairs
constexpr int kCombThreads = kQ * kTW / 2;  // combine warps: one pixel pair per thread
constexpr int kExtraThreads = kCombThreads + 32;  // + combine + loader
constexpr int kMaxThreads = kRoles * kMaxPairs * kItemsPerPair + kExtraThreads;
constexpr size_t kSmemLimit = 232448;          // 227 KB opt-in per block on sm_100
constexpr size_t kSmemPerSM = 233472;          // 228 KB per SM
constexpr size_t kSmemReservedPerBlock = 1024;

static_assert(kQ % kP == 0, "column-pass row groups tile the step");

#ifdef FBF_PHASES
// dev instrumentation: per-role cycle counters (thread 0 of each role)
__device__ unsigned long long g_phase_cycles[16];
__device__ unsigned long long g_cta_cycles[1024];
#define FBF_PHASE_T0() long long _ph_t = clock64()
#define FBF_PHASE(i)                                                        \
    do {                                                                    \
        if (tid == 0) {                                                     \
            long long _n = clock64();                                       \
            atomicAdd(&g_phase_cycles[i], (unsigned long long)(_n - _ph_t)); \
            _ph_t = _n;                                                     \
        }                                                                   \
    } while (0)
#else
#define FBF_PHASE_T0()
#define FBF_PHASE(i)
#endif

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
    unsigned int* bad_pixels;    // set to 1 if any output pixel's f is non-finite or outside [0, range_max]
    float range_max;             // R (filter.cpp:19-23 validation, fused into the combine)
    int width, height, n_frames, border;
    int out_row0, out_rows;
    int k_lo, n_pairs;           // chunk: k in [k_lo, k_lo + (k_lo == 0) + NKR)
    int k_first;                 // first k >= 1 of the chunk
    int first_chunk, last_chunk;
    int n_strips;
    int use_tma;                 // interior f tiles through the TMA bulk-copy engine
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
    static constexpr int RBP = RB + 1;                           // + the block the next row pass writes
    static constexpr int RROWS = RBP * kQ;                       // ring rows (private to a pair warp)
    static constexpr int RS = kTW + 2;                           // ring stride (float2), RS/2 odd
    static constexpr int NFS = 3;                                // f staging buffers (loader runs ahead)
#ifndef FBF_NGB
#define FBF_NGB 2
#endif
    static constexpr int NGB = FBF_NGB;                          // gen buffers (gen runs ahead)
    static constexpr int NCB = 2;                                // column-result buffers
    static constexpr size_t fstage_bytes = sizeof(float) * NFS * kQ * FSW;  // multiple of 128
    static constexpr size_t bar_bytes = 8 * (2 * NFS + 2 * NGB + 2 * NCB) + 8;  // mbarriers + counter
    static constexpr size_t misc_bytes = (bar_bytes + 127) / 128 * 128;
    static constexpr size_t fixed_bytes = fstage_bytes + misc_bytes;
    static constexpr size_t pair_bytes = sizeof(float2) * (size_t)(NGB * kQ * GS + NCB * kQ * kTW + RROWS * RS);
    static constexpr size_t smem_bytes(int pairs) { return fixed_bytes + pair_bytes * pairs; }
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

// Complex rotation z * w with packed FP32: t = z.x (w.x, w.y); z' = z.y (-w.y, w.x) + t,
// u = (-w.y, w.x) precomputed. gen and combine share this exact sequence.
__device__ __forceinline__ float2 cmul_rot(float2 z, float2 w, float2 u) {
    return __ffma2_rn(make_float2(z.y, z.y), u, __fmul2_rn(make_float2(z.x, z.x), w));
}
__device__ __forceinline__ float2 harmonic1c(float f, float inv_period) {
    float t = f * inv_period;
    t -= rintf(t);
    float sn, cs;
    __sincosf(t * 6.28318530717958647692f, &sn, &cs);
    return make_float2(cs, sn);
}
__device__ __forceinline__ float2 harmonic_firstc(float2 w, float2 u, int k_first) {
    float2 z = w;
    for (int k = 1; k < k_first; ++k) z = cmul_rot(z, w, u);
    return z;
}

// Packed forms for two adjacent pixels: (C, S) hold the two pixels' cosines and
// sines, per-lane arithmetic identical to rotate() / harmonic1().
struct CS2 {
    float2 c, s;
};
__device__ __forceinline__ CS2 harmonic1x2(float2 f, float inv_period) {
    float2 t = __fmul2_rn(f, make_float2(inv_period, inv_period));
    t = make_float2(t.x - rintf(t.x), t.y - rintf(t.y));
    t = __fmul2_rn(t, make_float2(6.28318530717958647692f, 6.28318530717958647692f));
    CS2 r;
    __sincosf(t.x, &r.s.x, &r.c.x);
    __sincosf(t.y, &r.s.y, &r.c.y);
    return r;
}
__device__ __forceinline__ CS2 rotate2(CS2 v, CS2 w, float2 nws) {  // nws = -w.s
    CS2 r;
    r.c = __ffma2_rn(v.c, w.c, __fmul2_rn(v.s, nws));
    r.s = __ffma2_rn(v.s, w.c, __fmul2_rn(v.c, w.s));
    return r;
}
__device__ __forceinline__ CS2 harmonic_first2(CS2 c1, int k_first) {
    const float2 nws = make_float2(-c1.s.x, -c1.s.y);
    CS2 cs = c1;
    for (int k = 1; k < k_first; ++k) cs = rotate2(cs, c1, nws);
    return cs;
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
__device__ __forceinline__ void cp_async16(float* smem_dst, const float* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem_dst)), "l"(gsrc));
}
// arrive-on of `bar` triggered when this thread's prior cp.async copies land
// (the pending count is incremented now and decremented on completion)
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
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
// raise the expected transaction bytes of the current phase (no arrival)
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// Blocking wait for the phase with the given parity. The suspend-time hint lets
// the hardware park the warp until the phase completes instead of spinning
// (a spinning try_wait loop costs issue slots the FFMA2 warps need).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000u)
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

// Vertical pass for output rows [Q0, Q0 + kP) of global step g. The window
// rows j in [Q0 - 2R, Q0 + kP) (relative to block g) resolve to (block, row)
// at compile time, so every load is a fixed offset from one of RB block pointers.
template <int R, int Q0>
__device__ __forceinline__ void column_pass(const float2* __restrict__ ring_pair, int blk, int x,
                                            const float* taps, float* out_col) {
    using G = Geometry<R>;
    constexpr int RB = G::RB, RS = G::RS;
    const float2* bptr[RB];
#pragma unroll
    for (int b = 0; b < RB; ++b) {  // bptr[b] = block (blk - b) mod RB
        int bb = blk - b;
        bb += bb < 0 ? RB : 0;
        bptr[b] = ring_pair + bb * kQ * RS + x;
    }
    float2 acc[kP];
#pragma unroll
    for (int o = 0; o < kP; ++o) acc[o] = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < kP + 2 * R; ++i) {
        const int j = Q0 + i - 2 * R;                     // compile-time
        const int b = j >= 0 ? 0 : (-j + kQ - 1) / kQ;    // blocks back
        const float2 v = bptr[b][(j + b * kQ) * RS];
#pragma unroll
        for (int o = 0; o < kP; ++o) {
            const int d = i - o;
            if (d >= 0 && d <= 2 * R) acc[o] = ffma2(v, taps[d >= R ? d - R : R - d], acc[o]);
        }
    }
#pragma unroll
    for (int o = 0; o < kP; ++o) {  // planar: [q][component][TW]
        float* oc = out_col + (Q0 + o) * 2 * kTW;
        oc[0] = acc[o].x;
        oc[kTW] = acc[o].y;
    }
}

// One software-pipelined pair-warp iteration: the horizontal pass of step t
// (DO_ROW; lane = (row q, 8-column chunk)) interleaved with the vertical pass of
// step t-1 (DO_COL; lane = column). The two FFMA2 streams are independent, so each
// hides the other's shared-memory latency. Row loads: (8+2R)/2 float4, column
// loads: 8+2R float2 -- always 2 column rows per row chunk.
template <int R, bool DO_ROW, bool DO_COL>
__device__ __forceinline__ void pair_iter(const float4* __restrict__ gin, float2* ring_pair, int blk_row,
                                          int blk_col, int lane, const float* taps, float* out_col,
                                          uint64_t* gen_empty_bar) {
    using G = Geometry<R>;
    constexpr int RB = G::RB, RBP = G::RBP, RS = G::RS;
    const int q = lane % kQ, xc = lane / kQ;
    float2 accr[kP], accc[kP];
    const float2* bptr[RB];
#pragma unroll
    for (int o = 0; o < kP; ++o) {
        accr[o] = make_float2(0.f, 0.f);
        accc[o] = make_float2(0.f, 0.f);
    }
    if (DO_COL) {
#pragma unroll
        for (int b = 0; b < RB; ++b) {  // bptr[b] = block (blk_col - b) mod RBP
            int bb = blk_col - b;
            bb += bb < 0 ? RBP : 0;
            bptr[b] = ring_pair + bb * kQ * RS + lane;
        }
    }
#pragma unroll
    for (int j = 0; j < (kP + 2 * R) / 2; ++j) {
        if (DO_ROW) {
            const float4 v4 = gin[j];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int jj = 2 * j + h;
                const float2 v = h ? make_float2(v4.z, v4.w) : make_float2(v4.x, v4.y);
#pragma unroll
                for (int o = 0; o < kP; ++o) {
                    const int d = jj - o;  // tap index 0..2R, ascending per output
                    if (d >= 0 && d <= 2 * R) accr[o] = ffma2(v, taps[d >= R ? d - R : R - d], accr[o]);
                }
            }
        }
        if (DO_COL) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int i = 2 * j + h;
                const int jr = i - 2 * R;                       // window row, compile-time
                const int b = jr >= 0 ? 0 : (-jr + kQ - 1) / kQ;  // blocks back
                const float2 v = bptr[b][(jr + b * kQ) * RS];
#pragma unroll
                for (int o = 0; o < kP; ++o) {
                    const int d = i - o;
                    if (d >= 0 && d <= 2 * R) accc[o] = ffma2(v, taps[d >= R ? d - R : R - d], accc[o]);
                }
            }
        }
    }
    if (DO_ROW) {
        __syncwarp();
        if (lane == 0) mbar_arrive(gen_empty_bar);  // this warp's gen rows consumed
        float4* hout = reinterpret_cast<float4*>(ring_pair + ((size_t)blk_row * kQ + q) * RS + xc * kP);
#pragma unroll
        for (int o = 0; o < kP / 2; ++o)
            hout[o] = make_float4(accr[2 * o].x, accr[2 * o].y, accr[2 * o + 1].x, accr[2 * o + 1].y);
    }
    if (DO_COL) {
#pragma unroll
        for (int o = 0; o < kP; ++o) {  // planar: [q][component][TW]
            float* oc = out_col + o * 2 * kTW + lane;
            oc[0] = accc[o].x;
            oc[kTW] = accc[o].y;
        }
    }
}

// Warp roles (np = channel pairs of the launch):
//   PAIR (np warps) : warp p owns channel pair p: horizontal pass of the step's
//                     Q rows into ITS OWN ring, then the vertical pass of the step
//                     from that ring into a column buffer -- no cross-warp handoff
//                     between the two passes
//   GEN  (np warps) : channel pairs of the next step into one of 2 gen buffers
//   COMB (4 warps)  : combine + divide, one output pixel pair per thread
//   LOAD (1 warp)   : f tiles into one of 3 staging buffers
// Handoffs GEN -> PAIR -> COMB and LOAD -> GEN are full/empty mbarrier pairs
// with per-warp arrivals, so no role waits for a sibling warp.

// Per-segment geometry shared by every role.
struct Segment {
    int frame, x0, ya, yb, a0, steps;
};

template <int R, int NKR>
__global__ void __launch_bounds__(kRoles * (1 + 2 * NKR) * kItemsPerPair + kExtraThreads, 1)
    fbf_fused_kernel(const __grid_constant__ Params p) {
    using G = Geometry<R>;
    constexpr int GW = G::GW, GS = G::GS, FSW = G::FSW, RB = G::RB, RBP = G::RBP, RROWS = G::RROWS, RS = G::RS;
    constexpr int NFS = G::NFS, NGB = G::NGB, NCB = G::NCB;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int np = p.n_pairs;
    float* fstage = reinterpret_cast<float*>(smem_raw);                         // [NFS][Q][FSW]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + G::fstage_bytes);
    uint64_t* fs_full = bars;                                // [NFS] LOAD -> GEN
    uint64_t* fs_empty = fs_full + NFS;                      // [NFS] GEN  -> LOAD
    uint64_t* gen_full = fs_empty + NFS;                     // [NGB] GEN  -> PAIR
    uint64_t* gen_empty = gen_full + NGB;                    // [NGB] PAIR -> GEN
    uint64_t* col_full = gen_empty + NGB;                    // [NCB] PAIR -> COMB
    uint64_t* col_empty = col_full + NCB;                    // [NCB] COMB -> PAIR
    unsigned int* s_fallbacks = reinterpret_cast<unsigned int*>(col_empty + NCB);
    float2* gen = reinterpret_cast<float2*>(smem_raw + G::fstage_bytes + G::misc_bytes);  // [NGB][np][Q][GS]
    float* colout = reinterpret_cast<float*>(gen + (size_t)NGB * np * kQ * GS);          // [NCB][np][Q][2][TW]
    float2* ring = reinterpret_cast<float2*>(colout + (size_t)NCB * np * kQ * 2 * kTW);  // [np][RROWS][RS]

    const int nrole = np * kItemsPerPair;  // threads of the PAIR and GEN roles
    // Warp slots: [PAIR | COMB | GEN | LOAD]; the scheduler favours higher warp ids,
    // so the latency-bound chains (GEN, COMB) get first pick of the issue slots and the
    // FFMA2 streams of the pair warps fill the rest.
    int role, tid;  // role: 0 GEN, 1 PAIR, 3 LOAD, 4 COMB
    {
        const int t = threadIdx.x;
        if (t < nrole)                          { role = 1; tid = t; }
        else if (t < nrole + kCombThreads)      { role = 4; tid = t - nrole; }
        else if (t < 2 * nrole + kCombThreads)  { role = 0; tid = t - nrole - kCombThreads; }
        else                                    { role = 3; tid = t - 2 * nrole - kCombThreads; }
    }
    const int lane = threadIdx.x & 31;
    const int zk = p.k_lo == 0 ? 1 : 0;  // k = 0 contributes the single pair (f, 1)
    if (threadIdx.x == 0) {
        *s_fallbacks = 0u;
        // every warp arrives on its own (no intra-role barrier): counts = warps
        const unsigned nw = (unsigned)np, ncw = kCombThreads / 32;
        for (int b = 0; b < NFS; ++b) { mbar_init(&fs_full[b], 1); mbar_init(&fs_empty[b], nw); }
        for (int b = 0; b < NGB; ++b) { mbar_init(&gen_full[b], nw); mbar_init(&gen_empty[b], nw); }
        for (int b = 0; b < NCB; ++b) { mbar_init(&col_full[b], nw); mbar_init(&col_empty[b], ncw); }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
#ifdef FBF_PHASES
    const long long _cta_t0 = clock64();
    unsigned long long _gt0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_gt0));
#endif

    // this CTA's contiguous share of the (frame, strip, row) units
    const long long U = p.total_units;
    const long long u_begin = U * blockIdx.x / gridDim.x;
    const long long u_end = U * (blockIdx.x + 1) / gridDim.x;
    const long long per_frame = (long long)p.n_strips * p.out_rows;
    // steps start e rows early so that output rows begin exactly at ya
    constexpr int e = (kQ - (2 * R) % kQ) % kQ;
    constexpr int s0 = (2 * R + e) / kQ;
    auto segment_at = [&](long long u, long long& next) {
        Segment sg;
        sg.frame = (int)(u / per_frame);
        const long long rem = u % per_frame;
        const int strip = (int)(rem / p.out_rows);
        const int row = (int)(rem % p.out_rows);
        const int len = (int)min((long long)(p.out_rows - row), u_end - u);
        next = u + len;
        sg.x0 = strip * kTW;
        sg.ya = p.out_row0 + row;
        sg.yb = sg.ya + len;
        sg.a0 = sg.ya - R - e;
        sg.steps = s0 + (len + kQ - 1) / kQ;
        return sg;
    };

    // ---- GEN: channel pairs of step s of segment sg into gen buffer gb --------------
    // item = it * nrole + tid covers the two adjacent pixels (q, xl), (q, xl + 1).
    constexpr int HGW = GW / 2;  // GW = TW + 2R is even
    constexpr int GITER = NKR > 0 ? (kQ * HGW + 2 * NKR * kItemsPerPair - 1) / (2 * NKR * kItemsPerPair)
                                  : (kQ * HGW + kItemsPerPair - 1) / kItemsPerPair;
    auto gen_step = [&](const Segment& sg, int s, int fb, int gb) {
        const int a = sg.a0 + s * kQ;
        const int xoff = (sg.x0 - R) - ((sg.x0 - R) & ~3);
        const float* fs = fstage + fb * kQ * FSW + xoff;
        float2* gbuf = gen + (size_t)gb * np * kQ * GS;
        const int lo = max(a, sg.ya - R), hi = min(a + kQ, sg.yb + R);
        const bool zb = p.border == 2;
        const float inv = p.inv_period;
#pragma unroll
        for (int it = 0; it < GITER; ++it) {
            const int item = it * nrole + tid;
            if (item < kQ * HGW) {
                const int q = item / HGW, xl = 2 * (item - q * HGW);
                const int gy = a + q, gx = sg.x0 - R + xl;
                const bool rowok = gy >= lo && gy < hi && (!zb || (gy >= 0 && gy < p.height));
                const bool va = rowok && (!zb || (gx >= 0 && gx < p.width));
                const bool vb = rowok && (!zb || (gx + 1 >= 0 && gx + 1 < p.width));
                const float2 f = make_float2(va ? fs[q * FSW + xl] : 0.f, vb ? fs[q * FSW + xl + 1] : 0.f);
                float4* gp = reinterpret_cast<float4*>(gbuf + q * GS + xl);
                if (zk) gp[0] = make_float4(f.x, va ? 1.f : 0.f, f.y, vb ? 1.f : 0.f);
                if (NKR > 0) {
                    const CS2 c1 = harmonic1x2(f, inv);
                    const float2 nws = make_float2(-c1.s.x, -c1.s.y);
                    CS2 cs = p.k_first > 1 ? harmonic_first2(c1, p.k_first) : c1;
                    if (!va) cs.c.x = cs.s.x = 0.f;
                    if (!vb) cs.c.y = cs.s.y = 0.f;
                    float4* gk = gp + (size_t)zk * kQ * GS / 2;
#pragma unroll
                    for (int kk = 0; kk < NKR; ++kk) {
                        const float2 cf = __fmul2_rn(cs.c, f), sf = __fmul2_rn(cs.s, f);
                        gk[(size_t)(2 * kk) * kQ * GS / 2] = make_float4(cf.x, sf.x, cf.y, sf.y);
                        gk[(size_t)(2 * kk + 1) * kQ * GS / 2] = make_float4(cs.c.x, cs.s.x, cs.c.y, cs.s.y);
                        if (kk + 1 < NKR) cs = rotate2(cs, c1, nws);
                    }
                }
            }
        }
    };

    // ---- COMB: combine of step s of segment sg from column buffer cb -----------------
    // one item = two adjacent output pixels per thread; f is re-read from the source
    // image (L2-resident) so nothing but the column results travels through smem
    auto combine_step = [&](const Segment& sg, int s, int cb) {
        const int a = sg.a0 + s * kQ;
        constexpr int HTW = kTW / 2;
        static_assert(kCombThreads == kQ * HTW, "one combine item per thread");
        const int q = tid / HTW, x = 2 * (tid - q * HTW);
        const int y = a - R + q, gxo = sg.x0 + x;
        if (y >= sg.yb || gxo >= p.width) return;
        const bool vb = gxo + 1 < p.width;
        const float* srow = p.src + (long long)sg.frame * p.src_frame_stride + (long long)(y - p.src_row0) * p.src_pitch;
        const float2 f = make_float2(__ldg(srow + gxo), vb ? __ldg(srow + gxo + 1) : 0.f);
        // validate_intensities (filter.cpp:19-23): every pixel is an output pixel exactly once
        if (p.bad_pixels && !(f.x >= 0.f && f.x <= p.range_max && f.y >= 0.f && f.y <= p.range_max))
            atomicOr(p.bad_pixels, 1u);
        float* dst = p.dst + (long long)sg.frame * p.dst_frame_stride;
        float2* acc = p.acc ? p.acc + (long long)sg.frame * p.acc_frame_stride : nullptr;
        float2 num = make_float2(0.f, 0.f), den = make_float2(0.f, 0.f);
        const long long ai = (long long)(y - p.out_row0) * p.width + gxo;
        if (!p.first_chunk) {
            const float2 nda = acc[ai], ndb = vb ? acc[ai + 1] : make_float2(0.f, 0.f);
            num = make_float2(nda.x, ndb.x);
            den = make_float2(nda.y, ndb.y);
        }
        // planar column results: [pair][q][component][TW]
        const float* go = colout + (size_t)cb * np * kQ * 2 * kTW + q * 2 * kTW + x;
        constexpr int PSTR = kQ * 2 * kTW;  // floats per pair
        if (zk) {
            const float2 gx0 = *reinterpret_cast<const float2*>(go);
            const float2 gy0 = *reinterpret_cast<const float2*>(go + kTW);
            const float2 c0 = make_float2(p.coeff[0], p.coeff[0]);
            num = __ffma2_rn(c0, gx0, num);
            den = __ffma2_rn(c0, gy0, den);
        }
        if (NKR > 0) {
            const CS2 c1 = harmonic1x2(f, p.inv_period);
            const float2 nws = make_float2(-c1.s.x, -c1.s.y);
            CS2 cs = p.k_first > 1 ? harmonic_first2(c1, p.k_first) : c1;
            const float* gk = go + zk * PSTR;
#pragma unroll
            for (int kk = 0; kk < NKR; ++kk) {
                const float2 ck = make_float2(p.coeff[zk + kk], p.coeff[zk + kk]);
                const float* gn = gk + (2 * kk) * PSTR;
                const float* gd = gk + (2 * kk + 1) * PSTR;
                const float2 gnx = *reinterpret_cast<const float2*>(gn);
                const float2 gny = *reinterpret_cast<const float2*>(gn + kTW);
                const float2 gdx = *reinterpret_cast<const float2*>(gd);
                const float2 gdy = *reinterpret_cast<const float2*>(gd + kTW);
                num = __ffma2_rn(ck, __ffma2_rn(cs.s, gny, __fmul2_rn(cs.c, gnx)), num);
                den = __ffma2_rn(ck, __ffma2_rn(cs.s, gdy, __fmul2_rn(cs.c, gdx)), den);
                if (kk + 1 < NKR) cs = rotate2(cs, c1, nws);
            }
        }
        float* drow = dst + (long long)(y - p.out_row0) * p.dst_pitch + gxo;
        if (p.last_chunk) {
            float oa = f.x, ob = f.y;
            unsigned nfb = 0;
            if (den.x > 1e-12f) oa = __fdividef(num.x, den.x); else ++nfb;
            if (den.y > 1e-12f) ob = __fdividef(num.y, den.y); else nfb += vb;
            if (nfb) atomicAdd(s_fallbacks, nfb);
            drow[0] = oa;
            if (vb) drow[1] = ob;
        } else {
            acc[ai] = make_float2(num.x, den.x);
            if (vb) acc[ai + 1] = make_float2(num.y, den.y);
        }
    };

    int gstep = 0;  // global step counter: buffers are used round-robin over it
    for (long long u = u_begin; u < u_end;) {
        long long next;
        const Segment sg = segment_at(u, next);
        u = next;
        const int steps = sg.steps;
        const int x0 = sg.x0, ya = sg.ya, yb = sg.yb, a0 = sg.a0;
        const int xs = (x0 - R) & ~3;  // f staging row origin (16-byte aligned)

        if (role == 3) {
            // ============================ LOAD ==============================
            // fstage row q holds f at columns [xs, xs + FSW), border-mapped with
            // 4-byte cp.async (or one TMA bulk copy per row for the in-image span,
            // FBF_STAGE=bulk). Zero-border rows/columns outside the image are never
            // read: GEN treats them as zero.
            const float* src = p.src + (long long)sg.frame * p.src_frame_stride;
            const int c0 = max(xs, 0), c1 = min(xs + FSW, p.width);  // in-image span
            const bool bulk = p.use_tma && c1 > c0;
            constexpr int LCOLS = (GW + 31) / 32;
            int lmx[LCOLS], loff[LCOLS];
            {
                const int wlo = x0 - R, whi = x0 + kTW + R;
                const int blo = bulk ? c0 : whi, bhi = bulk ? c1 : whi;  // bulk-covered span
                const int nleft = max(0, min(blo, whi) - wlo), nright = max(0, whi - max(bhi, wlo));
                const int ncols = bulk ? nleft + nright : GW;
#pragma unroll
                for (int j = 0; j < LCOLS; ++j) {
                    const int c = tid + 32 * j;
                    const int gx = bulk ? (c < nleft ? wlo + c : max(bhi, wlo) + (c - nleft)) : wlo + c;
                    lmx[j] = c < ncols ? map_border(gx, p.width, p.border) : -1;
                    loff[j] = gx - xs;
                }
            }
            for (int s = 0; s < steps; ++s) {
                const int g = gstep + s;
                const int fb = g % NFS;
                if (g >= NFS) mbar_wait(&fs_empty[fb], (unsigned)((g / NFS - 1) & 1));
                float* fs = fstage + fb * kQ * FSW;
                const int a = a0 + s * kQ;
                const int lo = max(a, ya - R), hi = min(a + kQ, yb + R);
#ifdef FBF_SKIP_LOAD
                if (tid == 0) mbar_arrive(&fs_full[fb]);
                continue;
#endif
                if (bulk) {
                    int nrows_src = 0;  // needed rows that read the image
                    for (int gy = lo; gy < hi; ++gy) nrows_src += map_border(gy, p.height, p.border) >= 0;
                    if (tid == 0 && nrows_src > 0)
                        mbar_expect_tx(&fs_full[fb], (unsigned)(sizeof(float) * (c1 - c0) * nrows_src));
                    __syncwarp();
                    if (tid < kQ) {
                        const int gy = a + tid;
                        const int my = (gy >= lo && gy < hi) ? map_border(gy, p.height, p.border) : -1;
                        if (my >= 0)
                            tma_bulk_g2s(fs + tid * FSW + (c0 - xs),
                                         src + (long long)(my - p.src_row0) * p.src_pitch + c0,
                                         (unsigned)(sizeof(float) * (c1 - c0)), &fs_full[fb]);
                    }
                }
#pragma unroll
                for (int q = 0; q < kQ; ++q) {
                    const int gy = a + q;
                    const int my = (gy >= lo && gy < hi) ? map_border(gy, p.height, p.border) : -1;
                    if (my < 0) continue;
                    const float* srow = src + (long long)(my - p.src_row0) * p.src_pitch;
#pragma unroll
                    for (int j = 0; j < LCOLS; ++j)
                        if (lmx[j] >= 0) cp_async4(fs + q * FSW + loff[j], srow + lmx[j]);
                }
                cp_async_mbar_arrive(&fs_full[fb]);
                __syncwarp();
                if (tid == 0) mbar_arrive(&fs_full[fb]);
            }
        } else if (role == 0) {
            // ============================= GEN ==============================
            FBF_PHASE_T0();
            for (int t = 0; t < steps; ++t) {
                const int g = gstep + t;
                const int fb = g % NFS, gb = g % NGB;
                FBF_PHASE(0);
                mbar_wait(&fs_full[fb], (unsigned)((g / NFS) & 1));
                if (g >= NGB) mbar_wait(&gen_empty[gb], (unsigned)((g / NGB - 1) & 1));
                FBF_PHASE(1);
#ifndef FBF_SKIP_GEN
                gen_step(sg, t, fb, gb);
#endif
                FBF_PHASE(4);
                __syncwarp();  // this warp's part of gen buffer gb written, fstage fb read
                if (lane == 0) {
                    mbar_arrive(&fs_empty[fb]);
                    mbar_arrive(&gen_full[gb]);
                }
                FBF_PHASE(5);
            }
        } else if (role == 4) {
            // ============================ COMB ==============================
            FBF_PHASE_T0();
            for (int sc = 0; sc < steps; ++sc) {
                const int g = gstep + sc;
                const int cb = g % NCB;
                mbar_wait(&col_full[cb], (unsigned)((g / NCB) & 1));
                FBF_PHASE(12);
#ifndef FBF_SKIP_COMB
                if (sc >= s0) combine_step(sg, sc, cb);
#endif
                FBF_PHASE(13);
                __syncwarp();  // this warp is done with column buffer cb
                if (lane == 0) mbar_arrive(&col_empty[cb]);
            }
        } else {
            // ============================= PAIR =============================
            // iteration t: horizontal pass of step t + vertical pass of step t - 1
            const int pr = tid / 32;  // this warp's channel pair
            float2* myring = ring + (size_t)pr * RROWS * RS;
            static_assert(kQ * (kTW / kP) == 32 && kQ == kP, "one pair = one warp");
            FBF_PHASE_T0();
            for (int t = 0; t <= steps; ++t) {
                const bool do_row = t < steps;
                const bool do_col = t >= 1 + s0;
                const int g = gstep + t, gc = g - 1;
                const int gb = g % NGB, cb = gc % NCB;
                FBF_PHASE(2);
                if (do_row) mbar_wait(&gen_full[gb], (unsigned)((g / NGB) & 1));
                // column buffer cb must have been consumed by COMB even on warm-up steps:
                // the arrival below completes a phase of col_full[cb], and a warp running
                // ahead must not complete the phase of a step its siblings have not finished
                if (t >= 1 && gc >= NCB) mbar_wait(&col_empty[cb], (unsigned)((gc / NCB - 1) & 1));
                FBF_PHASE(3);
                const float4* gin = reinterpret_cast<const float4*>(
                    gen + (((size_t)gb * np + pr) * kQ + lane % kQ) * GS + (lane / kQ) * kP);
                float* oc = colout + ((size_t)cb * np + pr) * kQ * 2 * kTW;
                const int blk_row = g % RBP, blk_col = gc % RBP;
                if (do_row && do_col)
                    pair_iter<R, true, true>(gin, myring, blk_row, blk_col, lane, p.taps, oc, &gen_empty[gb]);
                else if (do_row)
                    pair_iter<R, true, false>(gin, myring, blk_row, blk_col, lane, p.taps, oc, &gen_empty[gb]);
                else if (do_col)
                    pair_iter<R, false, true>(gin, myring, blk_row, blk_col, lane, p.taps, oc, &gen_empty[gb]);
                FBF_PHASE(6);
                __syncwarp();  // ring block / column results of this warp complete
                if (t >= 1 && lane == 0) mbar_arrive(&col_full[cb]);  // (warm-up steps hand over nothing)
                FBF_PHASE(11);
            }
        }
        gstep += steps;
    }
    __syncthreads();
#ifdef FBF_PHASES
    if (threadIdx.x == 0) {
        unsigned long long _gt1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_gt1));
        atomicMax(&g_phase_cycles[14], (unsigned long long)(clock64() - _cta_t0));
        atomicAdd(&g_phase_cycles[15], (unsigned long long)(clock64() - _cta_t0) * 1000ull / (_gt1 - _gt0 + 1));
        if (blockIdx.x < 1024) g_cta_cycles[blockIdx.x] = (unsigned long long)(clock64() - _cta_t0);
    }
#endif
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
    fbf_fused_kernel<R, NKR><<<grid, kRoles * p.n_pairs * kItemsPerPair + kExtraThreads, smem, stream>>>(p);
    return cudaGetLastError();
}

}  // namespace fbf_dev
