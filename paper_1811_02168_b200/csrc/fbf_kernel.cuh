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
// Dataflow (persistent CTAs, column strips streamed top to bottom, warp roles
// connected by mbarriers):
//   * The image is cut into strips of TW=32 output columns. Each CTA owns a
//     contiguous range of (frame, strip, row) units -- one or a few strip
//     segments -- so every CTA gets the same number of output rows.
//   * A segment is streamed in steps of Q input rows (Q = 16 for radii <= 16,
//     else 8; every FFMA2 lane produces P = Q outputs per pass).
//       LOAD : one warp stages f tiles (Q rows x (TW+2r) columns, border-mapped
//              through precomputed column maps) with 4-byte cp.async, up to two
//              steps ahead.
//       GEN  : channel pairs (f, 1) for k = 0 and (C_k f, S_k f), (C_k, S_k)
//              for k >= 1, with C_k + i S_k = exp(i k nu f) from one MUFU
//              sincos and the angle-addition recurrence, two pixels per thread
//              in packed FP32.
//       ROW  : one warp per channel pair: horizontal (2r+1)-tap pass, FFMA2
//              with the tap broadcast from a uniform register, into the pair's
//              ring of 1 + ceil(2r/Q) + 1 row blocks.
//       COL  : one warp per channel pair: vertical pass over the ring (window
//              offsets resolve at compile time) into a column-result tile.
//       COMB : num += c_k (C_k G(C_k f) + S_k G(S_k f)),
//              den += c_k (C_k G(C_k) + S_k G(S_k)) in ascending k, then
//              out = den > 1e-12 ? num / den : f; fallback count; the range
//              check of filter.cpp:19-23 on every output pixel's f.
//   * Channel pairs share taps, so one FFMA2 advances two channels (the
//     reference's 4K-2 channels are exactly 2K-1 pairs). Row and column passes
//     of a pair run in different warps so that the 2(2K-1) FFMA2 warps spread
//     evenly over the four SM sub-partitions (warp id mod 4).
//   * Coefficient chunks: when 2K-1 pairs do not fit in shared memory the
//     host launches one pass per chunk of k; (num, den) are carried in a
//     float2 scratch image between passes, still in ascending k.
#pragma once

#include <cuda.h>  // CUtensorMap (type only; the map is encoded on the host)
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <type_traits>

namespace fbf_dev {

constexpr int kTW = 32;          // output columns per strip
constexpr int kMaxKR = 4;        // k >= 1 terms per launch (template parameter NKR <= kMaxKR)
constexpr int kMaxPairs = 1 + 2 * kMaxKR;
constexpr int kMaxRadius = 32;
constexpr int kQ16MaxRadius = 16;  // Q = 16 steps are instantiated for r <= 16
#ifndef FBF_COMB_WARPS
#define FBF_COMB_WARPS 4
#endif
constexpr int kCombWarps = FBF_COMB_WARPS;
constexpr int kCombThreads = kCombWarps * 32;
#ifndef FBF_GEN_WARPS
#define FBF_GEN_WARPS 4
#endif
constexpr int kGenWarps = FBF_GEN_WARPS;
constexpr int kGenThreads = kGenWarps * 32;
constexpr int kExtraThreads = kCombThreads + kGenThreads + 32;  // combine + gen + loader
constexpr size_t kSmemLimit = 232448;          // 227 KB opt-in per block on sm_100
constexpr size_t kSmemPerSM = 233472;          // 228 KB per SM
constexpr size_t kSmemReservedPerBlock = 1024;

// Warp organisations of the FFMA2 work (template parameter M):
//   kPairMode : one warp per channel pair runs the row pass AND the (scatter)
//               column pass of a step -- no cross-warp handoff between passes
//               (r <= 16, where the 2r column partial sums fit in registers);
//   kSplitMode: one ROW and one COL warp per pair, connected by a ring of row
//               blocks -- twice the warps, so the FFMA2 work spreads more evenly
//               over the four SM sub-partitions (warp id mod 4).
//   kHalfMode : one ROW warp and two COL warps per pair; COL warp h produces
//               the output rows of parity h with R (not 2R) partial sums and
//               half the taps per row (same per-output order, same bits). The
//               3 np FFMA2 warps have weights 2:1:1, which the host places on
//               the sub-partitions so that each gets the same FFMA2 work
//               (Params::warp_role), for up to 7 pairs per launch.
//   kHalfWgMode: half mode with a fixed warpgroup layout and a setmaxnreg register
//               split (5 pairs, 24 warps; NKR = 2 only), see the kernel tail.
constexpr int kPairMode = 0, kSplitMode = 1, kHalfMode = 2, kHalfWgMode = 3;
__host__ __device__ constexpr bool is_half(int mode) { return mode == kHalfMode || mode == kHalfWgMode; }
// Pair mode with 7 pairs (16 warps): warpgroups 2-3 (7 pair warps + loader) run at
// FBF_REGSPLIT_HI registers, warpgroups 0-1 (gen + combine) at FBF_REGSPLIT_LO
// (setmaxnreg; 8 x LO + 8 x HI = 16 x 128). Measured on c1: 96/160 0.571 of the
// FMA peak vs 0.550 with the single 128-register layout (FBF_NO_REGSPLIT).
#ifndef FBF_REGSPLIT_LO
#define FBF_REGSPLIT_LO 96
#endif
#ifndef FBF_REGSPLIT_HI
#define FBF_REGSPLIT_HI 160
#endif
static_assert(FBF_REGSPLIT_LO + FBF_REGSPLIT_HI == 256, "8 warps at LO + 8 at HI must equal 16 warps at 128");
// kHalfWgMode (5 pairs, 24 warps at 80): gen + combine warpgroups at FBF_WG_LO, the rest at FBF_WG_HI
#ifndef FBF_WG_LO
#define FBF_WG_LO 64
#endif
#ifndef FBF_WG_HI
#define FBF_WG_HI 88
#endif
constexpr int kHalfMaxPairs = 7;
// threads of a launch: FFMA2 warps, plus combine, gen and loader (half mode:
// rounded up to whole sub-partition rows, unused slots idle)
__host__ __device__ constexpr int block_threads(int pairs, int mode) {
    return is_half(mode) ? 4 * ((3 * pairs + kGenWarps + kCombWarps + 1 + 3) / 4) * 32
                             : (mode == kPairMode ? 1 : 2) * 32 * pairs + kExtraThreads;
}
// Duo exchange region (appended to the larger rank's layout): [2 slots][Q * kTW / 2
// pixel pairs] float4 (num a, num b, den a, den b), then the slot barriers full[2], empty[2].
__host__ __device__ constexpr size_t duo_xchg_bytes(int q) { return 2 * (size_t)q * (kTW / 2) * 16 + 4 * 8; }
__host__ __device__ constexpr size_t align128(size_t v) { return (v + 127) / 128 * 128; }
enum Role { kRoleGen = 0, kRoleRow = 1, kRoleCol = 2, kRoleLoad = 3, kRoleComb = 4, kRoleIdle = 5 };


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
    int vec_ok;                  // rows are 16-byte aligned: interior tiles with 16-byte cp.async
    int ngb, ncb;                // gen / column-result buffers (1..2 each)
    long long total_units;       // n_frames * n_strips * out_rows
    float taps[kMaxRadius + 1];  // taps[j] = exp(-j^2 / (2 theta^2)), j = |d| (row pass)
    // the same taps for the column pass: a second copy keeps ptxas from hoisting
    // the shared values into ordinary registers when one warp runs both passes;
    // as separate kernel-parameter values each pass takes them as uniform-register
    // FFMA2 operands (measured: register operands cost FFMA2 issue rate)
    float taps_col[kMaxRadius + 1];
    float coeff[kMaxKR + 1];     // c_k of the chunk, ascending k
    float inv_period;            // 1 / (2T + 1)
    unsigned long long* prof;    // dev builds with FBF_PHASES: per warp slot [total, wait A, wait B, CTAs] cycles
    unsigned char warp_role[32]; // half mode: Role and role index of every warp slot
    unsigned char warp_idx[32];
    int use_tma2d;               // interior f tiles by the tensor map (kernel parameter `tmap`)
    int col_rounds;              // whole columns (frame, strip) per CTA taken round-robin before the tail
    int pdl;                     // host: launch with programmatic stream serialization
    // Duo launch (two coefficient chunks, no HBM scratch): clusters of 2 CTAs share each
    // work unit; rank r runs duo_chunk[r]. Rank 1 (the first chunk, k from 0) hands its
    // (num, den) partial sums per step to rank 0 (the last chunk) through distributed
    // shared memory; rank 0 continues from them exactly as the second launch of the
    // scratch path continues from the scratch image (same bits).
    int duo;
    struct ChunkSel {
        int k_lo, n_pairs, k_first;
        float coeff[kMaxKR + 1];
    } duo_chunk[2];
};

#ifdef FBF_PHASES
#define PWAIT(k, bar, par)                      \
    do {                                        \
        const long long _t0 = clock64();        \
        mbar_wait(bar, par);                    \
        _pw[k] += clock64() - _t0;              \
    } while (0)
// BAR.SYNC is deferred-blocking: an independent clock read right after it issues before
// the barrier completes (tools/microbench/bar_arrive.cu: 3 cycles reported for a 5000-cycle
// wait). The end time is therefore read behind a shared-memory load, which is ordered
// after the barrier.
#define PSYNC(k, id, n)                         \
    do {                                        \
        const long long _t0 = clock64();        \
        named_sync(id, n);                      \
        _pw[k] += clock_after_barrier() - _t0;  \
    } while (0)
#else
#define PWAIT(k, bar, par) mbar_wait(bar, par)
#define PSYNC(k, id, n) named_sync(id, n)
#endif

template <int R, int Q, int M>
struct Geometry {
    static_assert(Q == 8 || Q == 16, "step height");
    static constexpr bool PAIR = M == kPairMode;
    static constexpr int GW = kTW + 2 * R;                       // gen row width (pixels)
    static constexpr int GS = GW + ((2 - GW % 4) + 4) % 4;       // gen stride (float2), GS/2 odd
    static_assert(GS % 2 == 0, "gen pixel pairs are stored with 16-byte STS");
    static constexpr int FSW = (GW + 3 + 3) / 4 * 4;             // f staging row: GW + 16B-alignment slack
    // Column pass form: for R <= kScatterMaxRadius the 2R partial sums of a column
    // live in registers ("scatter": every row-pass output is read once), so the
    // ring is just a double buffer of Q rows; larger radii gather a window of
    // ring rows (RB blocks) per step.
    static constexpr bool SCATTER = R <= 16 || is_half(M);
    static_assert(SCATTER || !PAIR, "pair mode keeps the column partial sums in registers");
    static constexpr int RB = 1 + (2 * R + Q - 1) / Q;           // ring blocks a gather column pass reads
    static constexpr int RBN = SCATTER ? 1 : RB;                 // blocks a column pass reads
    // + the block the next row pass writes (split mode); pair mode: the warp's own
    // row pass of the next step starts after its column pass, one block suffices
    static constexpr int RBP = PAIR ? 1 : RBN + 1;
    static constexpr int RROWS = RBP * Q;                        // ring rows per pair
    static constexpr int RS = kTW + 1;                           // ring stride (float2), odd: conflict-free STS.64 across rows
#ifndef FBF_NFS
#define FBF_NFS 3
#endif
    static constexpr int NFS = FBF_NFS;                          // f staging buffers (loader runs ahead)
    static constexpr int kMaxBuf = 2;                            // gen / column buffers (named barrier ids)
    static constexpr size_t fstage_bytes = sizeof(float) * NFS * Q * FSW;  // multiple of 128
    static constexpr int n_bars = NFS + 2 * kMaxPairs * RBP;
    static constexpr size_t bar_bytes = 8 * n_bars + 8;          // mbarriers + counter
    static constexpr size_t misc_bytes = (bar_bytes + 127) / 128 * 128;
    static constexpr size_t fixed_bytes = fstage_bytes + misc_bytes;
    __host__ __device__ static constexpr size_t pair_bytes(int ngb, int ncb) {
        return sizeof(float2) * (size_t)(ngb * Q * GS + ncb * Q * kTW + RROWS * RS);
    }
    __host__ __device__ static constexpr size_t smem_bytes(int pairs, int ngb, int ncb) { return fixed_bytes + pair_bytes(ngb, ncb) * pairs; }
    static int max_pairs(int ngb, int ncb) {
        size_t budget = kSmemPerSM - kSmemReservedPerBlock;
        if (budget > kSmemLimit) budget = kSmemLimit;
        if (budget <= fixed_bytes) return 0;
        const size_t p = (budget - fixed_bytes) / pair_bytes(ngb, ncb);
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

// Packed forms for two adjacent pixels: (c, s) hold the two pixels' cosines and
// sines. exp(i (k+1) w) = exp(i k w) * exp(i w); gen and combine run this
// identical sequence, so modulation and demodulation factors agree bit for bit
// and do not depend on how k is split into chunks.
struct CS2 {
    float2 c, s;
};
// (cos, sin)(2 pi f / (2T+1)): turn reduction (exact: |t| < 1), then the MUFU
// pair on [-pi, pi].
__device__ __forceinline__ CS2 harmonic1x2(float2 f, float inv_period) {
    float2 t = __fmul2_rn(f, make_float2(inv_period, inv_period));
    t = make_float2(t.x - rintf(t.x), t.y - rintf(t.y));
    t = __fmul2_rn(t, make_float2(6.28318530717958647692f, 6.28318530717958647692f));
    CS2 r;
    __sincosf(t.x, &r.s.x, &r.c.x);
    __sincosf(t.y, &r.s.y, &r.c.y);
    return r;
}
// One rotation step, per component: C' = fma(-S, s, C c), S' = fma(C, s, S c).
// rotate2 works on two pixels packed per component, rotate1 on one pixel packed
// as (C, S) (one FMUL2 + one FFMA2 with a swapped, half-negated operand); both
// round identically, so gen (rotate1) and combine (rotate2) agree bit for bit.
__device__ __forceinline__ CS2 rotate2(CS2 v, CS2 w) {
    CS2 r;
    r.c = __ffma2_rn(make_float2(-v.s.x, -v.s.y), w.s, __fmul2_rn(v.c, w.c));
    r.s = __ffma2_rn(v.c, w.s, __fmul2_rn(v.s, w.c));
    return r;
}
__device__ __forceinline__ float2 rotate1(float2 z, float2 w) {
    return __ffma2_rn(make_float2(-z.y, z.x), make_float2(w.y, w.y), __fmul2_rn(z, make_float2(w.x, w.x)));
}
__device__ __forceinline__ CS2 harmonic_first2(CS2 c1, int k_first) {
    CS2 cs = c1;
    for (int k = 1; k < k_first; ++k) cs = rotate2(cs, c1);
    return cs;
}
__device__ __forceinline__ float2 harmonic_first1(float2 w, int k_first) {
    float2 z = w;
    for (int k = 1; k < k_first; ++k) z = rotate1(z, w);
    return z;
}

// float2 store to shared memory as st.shared.v2.f32: a plain float2 store through
// a generic pointer makes ptxas copy FMUL2/FFMA2 result pairs into a staging
// pair first (two MOVs per store, measured in the gen loop)
__device__ __forceinline__ void sts2(float2* p, float2 v) {
    // volatile keeps the order against the (volatile) barrier instructions that
    // publish the data; no memory clobber, so loads and math still schedule freely
    asm volatile("st.shared.v2.f32 [%0], {%1, %2};\n" ::"r"((unsigned)__cvta_generic_to_shared(p)), "f"(v.x), "f"(v.y));
}

// two adjacent float2 (16-byte aligned) as one st.shared.v4.f32
__device__ __forceinline__ void sts4(float2* p, float2 a, float2 b) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"((unsigned)__cvta_generic_to_shared(p)),
                 "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
}

// 1/x to ~1 ulp (MUFU.RCP); out = num / den has the same tolerance budget as
// __fdividef without its denormal-range fix-up instructions (den > 1e-12 here)
__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ float2 ffma2(float2 a, float w, float2 c) {
    return __ffma2_rn(a, make_float2(w, w), c);
}

// ---- synchronisation / async copy primitives -------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
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
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
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
// Duo exchange: wait on a local mbarrier whose arrivals come from the peer CTA
// (acquire at cluster scope, so the peer's distributed-shared-memory stores are visible)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAITC_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra WAITC_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000u)
        : "memory");
}
// arrive (release at cluster scope) on an mbarrier in the peer CTA's shared memory
__device__ __forceinline__ void mbar_arrive_remote(unsigned cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_addr) : "memory");
}

// Named CTA barriers for the warp-role handoffs: producers bar.arrive (no
// wait), consumers bar.sync -- a consumer warp blocked in bar.sync issues
// nothing, where an mbarrier try_wait loop keeps waking up (measured: the
// polling of idle gen/combine/loader warps cost about a third of all issued
// instructions). bar.arrive / bar.sync order shared-memory accesses among the
// participating threads.
__device__ __forceinline__ void named_arrive(int id, int nthreads) {
#ifdef FBF_DEV_PAIRONLY  // dev: FFMA2 warps alone, no handoffs (results invalid)
    return;
#endif
    asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int nthreads) {
#ifdef FBF_DEV_PAIRONLY
    return;
#endif
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ int lane_id_() { return (int)(threadIdx.x & 31); }
// dev (FBF_PHASES): clock read that cannot issue before a shared-memory load placed after
// a barrier has returned, i.e. before the barrier completed
__device__ __forceinline__ long long clock_after_barrier() {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const unsigned v = *reinterpret_cast<volatile unsigned*>(smem_raw);
    long long t;
    asm volatile(
        "{\n.reg .u32 z;\n.reg .u64 zz;\nand.b32 z, %1, 0;\ncvt.u64.u32 zz, z;\nmov.u64 %0, %%clock64;\nadd.u64 %0, %0, zz;\n}\n"
        : "=l"(t)
        : "r"(v)
        : "memory");
    return t;
}
// barrier ids (0 is __syncthreads): gen full/empty, column full/empty, f stage empty
constexpr int kBarGenFull = 1, kBarGenEmpty = 3, kBarColFull = 5, kBarColEmpty = 7, kBarFsEmpty = 9;
// ROW -> COL ring handoff of the half-mode rings (two blocks): one CTA-wide named
// barrier per ring block and direction, all pairs together (the ROW warps of all
// pairs do equal work). Per-pair mbarriers made the waiting COL warps poll: on c4
// their try_wait retry loop was 12 % of all issued instructions, issue slots the
// FFMA2 warps of the same sub-partition lost (c4 0.690 -> 0.703).
constexpr int kBarRingFull = 12, kBarRingEmpty = 14;

// 2-D tile of the 3-D tensor map (box FSW x Q x 1 at columns x.., rows y.. of frame
// z) into shared memory, completion on `bar` (coordinates outside the map fill 0).
__device__ __forceinline__ void tma_tile_g2s(float* smem_dst, const CUtensorMap* map, int x, int y, int z,
                                             uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
            smem_u32(smem_dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

// 1-D TMA bulk copy global -> shared (16-byte aligned, size multiple of 16),
// completion on `bar`.
__device__ __forceinline__ void tma_bulk_g2s(float* smem_dst, const float* gsrc, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(smem_dst)),
                 "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// Horizontal pass of one step for one channel pair: lane = (row q, chunk of Q
// columns); Q outputs per lane from (Q+2R)/2 LDS.128 of gen row q. Arrives on
// `gen_empty` once the gen rows are read, then writes the ring block.
template <int R, int Q>
__device__ __forceinline__ void row_pass(const float4* __restrict__ gin, float2* __restrict__ hout, const Params& pp,
                                         int gen_empty_id, int gen_threads) {
    float2 acc[Q];
#pragma unroll
    for (int o = 0; o < Q; ++o) acc[o] = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < (Q + 2 * R) / 2; ++j) {
        const float4 v4 = gin[j];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int jj = 2 * j + h;
            const float2 v = h ? make_float2(v4.z, v4.w) : make_float2(v4.x, v4.y);
#pragma unroll
            for (int o = 0; o < Q; ++o) {
                const int d = jj - o;  // tap index 0..2R, ascending per output
                if (d >= 0 && d <= 2 * R) acc[o] = ffma2(v, pp.taps[d >= R ? d - R : R - d], acc[o]);
            }
        }
    }
    named_arrive(gen_empty_id, gen_threads);  // this warp's gen rows consumed
#pragma unroll
    for (int o = 0; o < Q; ++o) hout[o] = acc[o];  // STS.64 straight from the accumulator pairs
}

// Vertical pass of ring block `blk` (the step's Q rows): lane = column, Q
// outputs from Q+2R ring rows. Window row jr (relative to the block's first row)
// resolves to (block, row) at compile time, so every load is a fixed offset
// from one of RB block pointers.
template <int R, int Q>
__device__ __forceinline__ void col_pass(const float2* __restrict__ ring_pair, int blk, int lane, const Params& pp,
                                         float2 (&acc)[Q]) {
    using G = Geometry<R, Q, kSplitMode>;
    constexpr int RB = G::RB, RBP = G::RBP, RS = G::RS;
    const float2* bptr[RB];
#pragma unroll
    for (int b = 0; b < RB; ++b) {  // bptr[b] = block (blk - b) mod RBP
        int bb = blk - b;
        bb += bb < 0 ? RBP : 0;
        bptr[b] = ring_pair + bb * Q * RS + lane;
    }
#pragma unroll
    for (int o = 0; o < Q; ++o) acc[o] = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < Q + 2 * R; ++i) {
        const int jr = i - 2 * R;                        // window row, compile-time
        const int b = jr >= 0 ? 0 : (-jr + Q - 1) / Q;   // blocks back
        const float2 v = bptr[b][(jr + b * Q) * RS];
#pragma unroll
        for (int o = 0; o < Q; ++o) {
            const int d = i - o;
            if (d >= 0 && d <= 2 * R) acc[o] = ffma2(v, pp.taps_col[d >= R ? d - R : R - d], acc[o]);
        }
    }
}

// Scatter form of the vertical pass for the Q rows of one ring block (lane =
// column). st[i] holds the partial sum of output row y - R + 1 + i after input
// row y; each new row v adds w(|d|) v to the 2R pending outputs while shifting
// them down one slot (one FFMA2 each, in place in ascending i), and completes
// output row y - R. Contributions enter every output in ascending input row,
// the reference's order (filter.cpp:52-70), so the result is bit-identical to
// the gather form.
template <int R, int Q>
__device__ __forceinline__ void col_scatter(const float2* __restrict__ hin, float2 (&st)[2 * R], float* out, bool store,
                                            const Params& pp) {
    constexpr int RS = kTW + 1;
#pragma unroll
    for (int r = 0; r < Q; ++r) {
        const float2 v = hin[r * RS];
        const float2 o = ffma2(v, pp.taps_col[R], st[0]);
#pragma unroll
        for (int i = 0; i < 2 * R - 1; ++i) {
            const int d = R - 1 - i;
            st[i] = ffma2(v, pp.taps_col[d >= 0 ? d : -d], st[i + 1]);
        }
        st[2 * R - 1] = __fmul2_rn(v, make_float2(pp.taps_col[R], pp.taps_col[R]));
        if (store) {  // planar: [channel][q][TW]
            out[r * kTW] = o.x;
            out[(Q + r) * kTW] = o.y;
        }
    }
}

// Half of the scatter column pass: output rows q of the step with q % 2 == H
// (q = r: the output completed by input row r). st[i] holds the partial sum of
// the i-th pending output of this parity: R of them. A completing row (r % 2 ==
// H) finishes st[0], shifts, and opens the output R rows below; the other rows
// add to all R pending outputs. Per output, contributions still enter in
// ascending input row from a product, so the bits equal col_scatter's.
template <int R, int Q, int H>
__device__ __forceinline__ void col_scatter_half(const float2* __restrict__ hin, float2 (&st)[R], float* out,
                                                 bool store, const Params& pp) {
    constexpr int RS = kTW + 1;
#pragma unroll
    for (int r = 0; r < Q; ++r) {
        const float2 v = hin[r * RS];
        if ((r & 1) == H) {
            const float2 o = ffma2(v, pp.taps_col[R], st[0]);
#pragma unroll
            for (int i = 0; i + 1 < R; ++i) {
                const int d = R - 2 * (i + 1);
                st[i] = ffma2(v, pp.taps_col[d >= 0 ? d : -d], st[i + 1]);
            }
            st[R - 1] = __fmul2_rn(v, make_float2(pp.taps_col[R], pp.taps_col[R]));
            if (store) {  // planar: [channel][q][TW]
                out[r * kTW] = o.x;
                out[(Q + r) * kTW] = o.y;
            }
        } else {
#pragma unroll
            for (int i = 0; i < R; ++i) {
                const int d = R - 1 - 2 * i;
                st[i] = ffma2(v, pp.taps_col[d >= 0 ? d : -d], st[i]);
            }
        }
    }
}

// Per-segment geometry shared by every role.
struct Segment {
    int frame, x0, ya, yb, a0, steps;
};

// Warp slots: [ROW np | COL np | COMB 4 | GEN np | LOAD 1]. Handoffs are
// full/empty mbarrier pairs with per-warp arrivals:
//   LOAD -fs-> GEN -gen-> ROW p -ring p-> COL p -col-> COMB
template <int R, int Q, int NKR, int M>
// `tmap`: 3-D tensor map over the source (columns, rows present in src, frames)
// with a box of one f tile (FSW, Q, 1) -- a kernel parameter of its own (its
// address is taken for the TMA; inside Params that made ptxas spill the FFMA2 loops).
__global__ void __launch_bounds__(block_threads(1 + 2 * NKR, M), 1)
    fbf_fused_kernel(const __grid_constant__ Params p, const __grid_constant__ CUtensorMap tmap) {
    using G = Geometry<R, Q, M>;
    constexpr int GW = G::GW, GS = G::GS, FSW = G::FSW, RB = G::RB, RBP = G::RBP, RROWS = G::RROWS, RS = G::RS;
    constexpr int NFS = G::NFS;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const bool duo = p.duo != 0;
    unsigned crank = 0;  // rank in the cluster (duo launches)
    if (duo) asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(crank));
    // this CTA's coefficient chunk
    const int np = duo ? p.duo_chunk[crank].n_pairs : p.n_pairs;
    const int k_lo = duo ? p.duo_chunk[crank].k_lo : p.k_lo;
    const int k_first = duo ? p.duo_chunk[crank].k_first : p.k_first;
    const float* coeff = duo ? p.duo_chunk[crank].coeff : p.coeff;
    // (num, den) carried between chunks: into the combine (scratch image or, duo rank 0,
    // the exchange slots), out of it (scratch or, duo rank 1, the peer's exchange slots)
    const bool x_in = duo && crank == 0, x_out = duo && crank == 1;
    const bool carry_in = duo ? x_in : !p.first_chunk;
    const bool last = duo ? x_in : p.last_chunk != 0;
    const int ngb = p.ngb, ncb = p.ncb;  // ngb, ncb in {1, 2}: buffer index = g & (n - 1)
    float* fstage = reinterpret_cast<float*>(smem_raw);                         // [NFS][Q][FSW]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + G::fstage_bytes);
    uint64_t* fs_full = bars;                                // [NFS] LOAD -> GEN (cp.async completion)
    uint64_t* ring_full = fs_full + NFS;                     // [np][RBP] ROW p -> COL p (split mode)
    uint64_t* ring_empty = ring_full + kMaxPairs * RBP;      // [np][RBP] COL p -> ROW p
    float2* gen = reinterpret_cast<float2*>(smem_raw + G::fixed_bytes);  // [ngb][np][Q][GS]
    float2* colout = gen + (size_t)ngb * np * Q * GS;                    // [ncb][np] x [2][Q][TW] floats
    float2* ring = colout + (size_t)ncb * np * Q * kTW;                  // [np][RROWS][RS]
    // duo exchange region, after the larger rank's layout (the same offset in both CTAs)
    const size_t xoff = duo ? align128(G::smem_bytes(max(p.duo_chunk[0].n_pairs, p.duo_chunk[1].n_pairs), p.ngb, p.ncb)) : 0;
    float4* xslot = reinterpret_cast<float4*>(smem_raw + xoff);              // [2][Q * kTW / 2]
    uint64_t* xbar = reinterpret_cast<uint64_t*>(smem_raw + xoff + 2 * (size_t)Q * (kTW / 2) * 16);  // full[2], empty[2]

    const int nrole = np * 32;  // threads of the ROW/PAIR role (and of the COL role in split mode)
    const int nf = G::PAIR ? nrole : 2 * nrole;  // FFMA2 threads
    int role, tid;  // Role; ROW is PAIR in pair mode
    if constexpr (is_half(M)) {
        const int w = (int)(threadIdx.x / 32);
        role = p.warp_role[w];
        tid = p.warp_idx[w] * 32 + (int)(threadIdx.x & 31);
    } else {
        // Roles are numbered from the LAST warp down: the FFMA2 warps get the highest
        // warp ids, which the issue arbiter of a sub-partition serves first; the
        // latency-bound roles (gen, combine, loader) have slack and fill the gaps.
        const int t = (blockDim.x / 32 - 1 - (int)(threadIdx.x / 32)) * 32 + (threadIdx.x & 31);
        constexpr int CG = kCombThreads + kGenThreads;
        if (t < nrole)                     { role = kRoleRow; tid = t; }
        else if (t < nf)                   { role = kRoleCol; tid = t - nrole; }
        else if (t < nf + kCombThreads)    { role = kRoleComb; tid = t - nf; }
        else if (t < nf + CG)              { role = kRoleGen; tid = t - nf - kCombThreads; }
        else if (t < nf + CG + 32)         { role = kRoleLoad; tid = t - nf - CG; }
        else                               { role = kRoleIdle; tid = 0; }  // duo rank with fewer pairs
#ifndef FBF_NO_REGSPLIT
        // register-split layout (pair mode, 7 pairs, 16 warps): warpgroups 2-3 hold the
        // 7 pair warps and the loader, 0-1 the combine and gen warps, so that every
        // role's code runs from one instance only (no duplicated hot code)
        if (M == kPairMode && NKR == 3 && blockDim.x == 512 && np == 7 && t >= nf) {
            const int w = (int)(threadIdx.x / 32);  // 0..8
            if (w == 8)     { role = kRoleLoad; tid = lane_id_(); }
            else if (w >= 4) { role = kRoleComb; tid = (7 - w) * 32 + lane_id_(); }
            else            { role = kRoleGen; tid = (3 - w) * 32 + lane_id_(); }
        }
#endif
    }
    const int lane = threadIdx.x & 31;
    const int zk = k_lo == 0 ? 1 : 0;  // k = 0 contributes the single pair (f, 1)
    // named-barrier thread counts: producers + consumers of each handoff
    const int gen_threads = kGenThreads + nrole;   // GEN -> ROW/PAIR and back
    const int col_threads = (is_half(M) ? 2 : 1) * nrole + kCombThreads;  // COL/PAIR -> COMB and back
    constexpr int kFsThreads = kGenThreads + 32;   // GEN -> LOAD (f stage empty)
    // Ring handoffs through named barriers (ROW + COL threads of all pairs), one id per
    // step parity and direction: half mode and the split-mode gather ring (r > 16).
    // ROW at step g waits for COL done with step g - 2 (the block it overwrites was last
    // read then: RBP - RB + 1 = 2), every step from g = 2 on so the phases pair up.
    // The split-mode scatter ring (c3) keeps the per-pair mbarriers: its 9-pair
    // launches measured 0.493 -> 0.489 with the CTA-wide barrier (the pairs lockstep).
#ifdef FBF_DEV_RING_MBAR_MAXR  // dev: half-mode rings through per-pair mbarriers up to this radius
    constexpr bool RING_NB = (is_half(M) && R > FBF_DEV_RING_MBAR_MAXR) || (M == kSplitMode && !G::SCATTER);
#else
    constexpr bool RING_NB = is_half(M) || (M == kSplitMode && !G::SCATTER);
#endif
    static_assert(!RING_NB || RBP - RB + 1 == 2 || RBP == 2, "ROW may run two steps ahead of COL");
    static_assert(kBarFsEmpty + NFS <= kBarRingFull, "named barrier ids overlap");
    const int ring_threads = (is_half(M) ? 3 : 2) * nrole;
#ifdef FBF_PHASES
    long long _pw[2] = {0, 0};
    const long long _pt0 = clock64();
#endif
    unsigned n_fallbacks = 0;  // combine threads: fallback pixels (filter.cpp:203-208)
    unsigned xstep = 0;        // combine threads, duo: output steps exchanged so far
    if (threadIdx.x == 0) {
        for (int b = 0; b < NFS; ++b) mbar_init(&fs_full[b], 1);
        for (int b = 0; b < np * RBP; ++b) {
            mbar_init(&ring_full[b], 1);
            mbar_init(&ring_empty[b], is_half(M) ? 2 : 1);  // both COL halves release a block
        }
        if (duo) {
            for (int b = 0; b < 4; ++b) mbar_init(&xbar[b], kCombThreads);  // full[2], empty[2]
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (duo) {  // the peer's exchange barriers are initialised before any remote arrive
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    } else {
        __syncthreads();
    }
    // Programmatic dependent launch: this grid may start while the previous kernel on
    // the stream drains (its CTAs free SMs at different times). Wait for that grid and
    // its memory (the previous chunk's (num, den) scratch, a caller's producer kernel)
    // before any global access, then let the next launch begin its own prologue.
    // Without the launch attribute both instructions are no-ops.
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");

    // This CTA's work: `col_rounds` whole columns (frame, strip) taken round-robin --
    // column j * gridDim.x + blockIdx.x in round j, so at any time the CTAs stream
    // neighbouring strips over the same rows and the halo columns two strips share
    // are read from DRAM once (L2 hits for the second) -- then a contiguous share of
    // the remaining (frame, strip, row) units.
    const long long U = p.total_units;
    // work shares: one per CTA, or per cluster of 2 in a duo launch (both ranks walk it)
    const int wid = duo ? (int)(blockIdx.x >> 1) : (int)blockIdx.x, nw = duo ? (int)(gridDim.x >> 1) : (int)gridDim.x;
    const long long tail0 = (long long)p.col_rounds * nw * p.out_rows;  // first unit of the tail
    const long long u_begin = tail0 + (U - tail0) * wid / nw;
    const long long u_end = tail0 + (U - tail0) * (wid + 1) / nw;
    const long long per_frame = (long long)p.n_strips * p.out_rows;
    // steps start e rows early so that output rows begin exactly at ya; the first
    // s0 steps of a segment only fill the ring
    constexpr int e = (Q - (2 * R) % Q) % Q;
    constexpr int s0 = (2 * R + e) / Q;
    static_assert(s0 == RB - 1, "warm-up steps fill all but one ring block");
    auto segment_at = [&](long long u, long long uend, long long& next) {
        Segment sg;
        sg.frame = (int)(u / per_frame);
        const long long rem = u % per_frame;
        const int strip = (int)(rem / p.out_rows);
        const int row = (int)(rem % p.out_rows);
        const int len = (int)min((long long)(p.out_rows - row), uend - u);
        next = u + len;
        sg.x0 = strip * kTW;
        sg.ya = p.out_row0 + row;
        sg.yb = sg.ya + len;
        sg.a0 = sg.ya - R - e;
        sg.steps = s0 + (len + Q - 1) / Q;
        return sg;
    };

    // ---- GEN: channel pairs of step s of segment sg into gen buffer gb --------------
    // item = it * kGenThreads + tid covers the two adjacent pixels (q, xl), (q, xl + 1).
    constexpr int HGW = GW / 2;  // GW = TW + 2R is even
    constexpr int GITER = (Q * HGW + kGenThreads - 1) / kGenThreads;
    // Per-thread item geometry is fixed over steps and segments: the f staging
    // offset (x0 - R is congruent to -R mod 4, so the staged row origin lies at a
    // compile-time offset XOFF), the gen offset, and the row q (-1: no item).
    constexpr int XOFF = ((-R) % 4 + 4) % 4;
    struct GenItem {
        int fso, go, q, cm;  // cm: bit 0/1 = pixel a/b lies in the image (or the border is not zero)
    };
    auto gen_items = [&](const Segment& sg, GenItem (&gi)[GITER]) {
        const bool zb = p.border == 2;
#pragma unroll
        for (int it = 0; it < GITER; ++it) {
            const int item = it * kGenThreads + tid;
            const int q = item / HGW, xl = 2 * (item - q * HGW);
            const int gx = sg.x0 - R + xl;
            const int cm = (!zb || (gx >= 0 && gx < p.width) ? 1 : 0) | (!zb || (gx + 1 >= 0 && gx + 1 < p.width) ? 2 : 0);
            gi[it] = GenItem{q * FSW + xl + XOFF, q * GS + xl, item < Q * HGW ? q : -1, cm};
        }
    };
    auto gen_step = [&](const Segment& sg, int s, int fb, int gb, const GenItem (&gi)[GITER]) {
        const int a = sg.a0 + s * Q;
        const float* fs = fstage + fb * Q * FSW;
        float2* gbuf = gen + gb * np * Q * GS;
        // rows of the step that feed an output row and (zero border) lie in the image
        int lo = max(a, sg.ya - R), hi = min(a + Q, sg.yb + R);
        if (p.border == 2) {
            lo = max(lo, 0);
            hi = min(hi, p.height);
        }
        const unsigned nrows = (unsigned)max(hi - lo, 0);
        const float inv = p.inv_period;
        const bool kfirst = k_first > 1;
        // MASKED: zero border -- pixels outside the image and rows outside the needed
        // window contribute exact zeros. Symmetric / replicate borders map every staged
        // pixel into the image, and rows outside [lo, hi) (stale stage data) only reach
        // output rows that are never stored: each output's column sum opens fresh R rows
        // above it (col_scatter) and the combine writes rows [ya, yb) only -- so the
        // unmasked body skips the selects.
        auto body = [&](auto masked_c) {
            constexpr bool MASKED = decltype(masked_c)::value;
#pragma unroll 2
            for (int it = 0; it < GITER; ++it) {
                const int q = gi[it].q;
                if (q >= 0) {
                    // unconditional loads (rows the loader skipped hold stale values), then select
                    const float fa = fs[gi[it].fso], fbv = fs[gi[it].fso + 1];
                    bool va = true, vb = true;
                    if constexpr (MASKED) {
                        const bool rowok = (unsigned)(a + q - lo) < nrows;
                        va = rowok && (gi[it].cm & 1);
                        vb = rowok && (gi[it].cm & 2);
                    }
                    const float2 f = MASKED ? make_float2(va ? fa : 0.f, vb ? fbv : 0.f) : make_float2(fa, fbv);
                    // per pixel (first, second) channel pairs, stored as float2 at gp[0] / gp[1]
                    float2* gp = gbuf + gi[it].go;
                    if (zk) {
                        sts4(gp, make_float2(f.x, MASKED && !va ? 0.f : 1.f), make_float2(f.y, MASKED && !vb ? 0.f : 1.f));
                    }
                    if (NKR > 0) {
                        const CS2 h = harmonic1x2(f, inv);
                        const float2 w0 = make_float2(h.c.x, h.s.x), w1 = make_float2(h.c.y, h.s.y);
                        float2 z0 = kfirst ? harmonic_first1(w0, k_first) : w0;
                        float2 z1 = kfirst ? harmonic_first1(w1, k_first) : w1;
                        if constexpr (MASKED) {
                            if (!va) z0 = make_float2(0.f, 0.f);
                            if (!vb) z1 = make_float2(0.f, 0.f);
                        }
                        float2* gk = gp + zk * (Q * GS);
#pragma unroll
                        for (int kk = 0; kk < NKR; ++kk) {
                            float2* pf = gk + (2 * kk) * (Q * GS);      // (C_k f, S_k f)
                            float2* pc = gk + (2 * kk + 1) * (Q * GS);  // (C_k, S_k)
                            // both pixels' pairs in one STS.128 (gp is 16-byte aligned: GS, xl even)
                            sts4(pf, __fmul2_rn(z0, make_float2(f.x, f.x)), __fmul2_rn(z1, make_float2(f.y, f.y)));
                            sts4(pc, z0, z1);
                            if (kk + 1 < NKR) {
                                z0 = rotate1(z0, w0);
                                z1 = rotate1(z1, w1);
                            }
                        }
                    }
                }
            }
        };
        if (p.border == 2) body(std::true_type{});
        else body(std::false_type{});
    };

    // ---- COMB: combine of step s of segment sg from column buffer cb -----------------
    // one item = two adjacent output pixels; f is re-read from the source image
    // (L2-resident) so nothing but the column results travels through smem
    constexpr int HTW = kTW / 2;
    constexpr int CITER = Q * HTW / kCombThreads;
    static_assert(CITER * kCombThreads == Q * HTW, "combine items tile the step");
    // Per-thread items: pointers to the item's pixels in the first output step
    // of the segment, advanced by Q rows per step.
    struct CombItem {
        const float* sp;  // f
        float* dp;        // output
        float2* ap;       // (num, den) scratch
        int co;           // column-result offset (float2) within a pair's tile
        int y;            // output row of the current step
        bool colok, vb;   // pixel pair in the image / second pixel in the image
    };
    auto comb_items = [&](const Segment& sg, CombItem (&ci)[CITER]) {
#pragma unroll
        for (int it = 0; it < CITER; ++it) {
            const int item = it * kCombThreads + tid;
            const int q = item / HTW, x = 2 * (item - q * HTW);
            const int gxo = sg.x0 + x, y = sg.a0 + s0 * Q - R + q;
            ci[it].co = q * kTW + x;
            ci[it].y = y;
            ci[it].colok = gxo < p.width;
            ci[it].vb = gxo + 1 < p.width;
            ci[it].sp = p.src + (long long)sg.frame * p.src_frame_stride + (long long)(y - p.src_row0) * p.src_pitch + gxo;
            ci[it].dp = p.dst + (long long)sg.frame * p.dst_frame_stride + (long long)(y - p.out_row0) * p.dst_pitch + gxo;
            ci[it].ap = p.acc ? p.acc + (long long)sg.frame * p.acc_frame_stride + (long long)(y - p.out_row0) * p.width + gxo
                              : nullptr;
        }
    };
    // f of the step's output pixels, loaded before the step's column results are
    // waited for so that the L2 latency overlaps the wait
    // (and, after the first coefficient chunk, the (num, den) carried in the scratch
    // image: an HBM read whose latency otherwise stalls the step, c2 0.585 -> 0.595)
    auto combine_load = [&](const Segment& sg, const CombItem (&ci)[CITER], float2 (&fv)[CITER],
                            float4 (&nd)[CITER]) {
#pragma unroll
        for (int it = 0; it < CITER; ++it) {
            fv[it] = make_float2(0.f, 0.f);
            nd[it] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (ci[it].y < sg.yb && ci[it].colok) {
                fv[it] = make_float2(__ldg(ci[it].sp), ci[it].vb ? __ldg(ci[it].sp + 1) : 0.f);
                if (carry_in && !x_in) {
                    const float2 a = __ldcg(ci[it].ap), b = ci[it].vb ? __ldcg(ci[it].ap + 1) : make_float2(0.f, 0.f);
                    nd[it] = make_float4(a.x, b.x, a.y, b.y);  // (num a, num b, den a, den b)
                }
            }
        }
    };
    // per-step pointer advances (64-bit adds, no wide multiplies in the step loop)
    const long long src_step = (long long)Q * p.src_pitch, dst_step = (long long)Q * p.dst_pitch,
                    acc_step = (long long)Q * p.width;
    auto combine_step = [&](const Segment& sg, int cb, CombItem (&ci)[CITER], const float2 (&fv)[CITER],
                            const float4 (&nd)[CITER], unsigned xdst) {
        const float* cbase = reinterpret_cast<const float*>(colout + cb * np * Q * kTW);
        const bool kfirst_c = k_first > 1;
#pragma unroll
        for (int it = 0; it < CITER; ++it) {
            CombItem& c = ci[it];
            if (c.y < sg.yb && c.colok) {
                const bool vb = c.vb;
                const float2 f = fv[it];
                // validate_intensities (filter.cpp:19-23): every pixel is an output pixel exactly once
                if (p.bad_pixels && !(f.x >= 0.f && f.x <= p.range_max && f.y >= 0.f && f.y <= p.range_max))
                    atomicOr(p.bad_pixels, 1u);
                float2 num = make_float2(0.f, 0.f), den = make_float2(0.f, 0.f);
                if (carry_in) {
                    num = make_float2(nd[it].x, nd[it].y);
                    den = make_float2(nd[it].z, nd[it].w);
                }
                // planar column results [pair][channel][q][TW]: float2 = the two pixels of one channel
                const float2* go = reinterpret_cast<const float2*>(cbase + c.co);
                constexpr int CSTR = Q * kTW / 2;  // float2 per channel plane
                // ZK (chunk holds k = 0) as a compile-time constant: coefficient and
                // column-tile offsets become immediates
                auto accumulate = [&](auto zkc) {
                    constexpr int ZK = decltype(zkc)::value;
                    if (ZK) {
                        const float2 c0 = make_float2(coeff[0], coeff[0]);
                        num = __ffma2_rn(c0, go[0], num);
                        den = __ffma2_rn(c0, go[CSTR], den);
                    }
                    if (NKR > 0) {
                        const CS2 c1 = harmonic1x2(f, p.inv_period);
                        CS2 cs = kfirst_c ? harmonic_first2(c1, k_first) : c1;
                        const float2* gk = go + ZK * 2 * CSTR;
#pragma unroll
                        for (int kk = 0; kk < NKR; ++kk) {
                            const float2 ck = make_float2(coeff[ZK + kk], coeff[ZK + kk]);
                            const float2* pn = gk + (4 * kk) * CSTR;  // G(C_k f), G(S_k f)
                            const float2* pd = pn + 2 * CSTR;         // G(C_k), G(S_k)
                            num = __ffma2_rn(ck, __ffma2_rn(cs.s, pn[CSTR], __fmul2_rn(cs.c, pn[0])), num);
                            den = __ffma2_rn(ck, __ffma2_rn(cs.s, pd[CSTR], __fmul2_rn(cs.c, pd[0])), den);
                            if (kk + 1 < NKR) cs = rotate2(cs, c1);
                        }
                    }
                };
                if (zk) accumulate(std::integral_constant<int, 1>{});
                else accumulate(std::integral_constant<int, 0>{});
                if (last) {
                    float oa = f.x, ob = f.y;
                    unsigned nfb = 0;
                    if (den.x > 1e-12f) oa = num.x * rcp_approx(den.x); else ++nfb;
                    if (den.y > 1e-12f) ob = num.y * rcp_approx(den.y); else nfb += vb;
                    n_fallbacks += nfb;
                    c.dp[0] = oa;
                    if (vb) c.dp[1] = ob;
                } else if (x_out) {  // into the peer's exchange slot (distributed shared memory)
                    asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(
                                     xdst + (unsigned)(it * kCombThreads + tid) * 16u),
                                 "f"(num.x), "f"(num.y), "f"(den.x), "f"(den.y)
                                 : "memory");
                } else {
                    c.ap[0] = make_float2(num.x, den.x);
                    if (vb) c.ap[1] = make_float2(num.y, den.y);
                }
            }
            c.y += Q;
            c.sp += src_step;
            c.dp += dst_step;
            if (p.acc) c.ap += acc_step;
        }
    };

    // Per-role segment loops: each role walks this CTA's segments on its own, so a
    // role's loop carries only its own state across segments (one shared segment
    // loop kept every role's loop state live in every role; measured c4 0.638 -> 0.650).
    auto for_each_segment = [&](auto&& body) {
        int gstep = 0;  // global step counter: buffers and ring blocks are used round-robin over it
        int j = 0;      // round of the whole-column part
        for (long long u = u_begin;;) {
            // one call site of `body` (two loops would inline every role twice)
            long long next, a, b;
            if (j < p.col_rounds) {
                a = ((long long)j++ * nw + wid) * p.out_rows;
                b = a + p.out_rows;
            } else if (u < u_end) {
                a = u;
                b = u_end;
            } else {
                break;
            }
            const Segment sg = segment_at(a, b, next);
            if (a == u) u = next;
            body(sg, gstep);
            gstep += sg.steps;
        }
    };
#define FBF_SEGMENT_LOCALS                                          \
    const int steps = sg.steps;                                     \
    const int x0 = sg.x0, ya = sg.ya, yb = sg.yb, a0 = sg.a0;       \
    const int xs = (x0 - R) & ~3; /* f staging row origin (16-byte aligned) */ \
    (void)steps, (void)x0, (void)ya, (void)yb, (void)a0, (void)xs;

    auto run_roles = [&](auto fma_region) {
    constexpr bool FMA = decltype(fma_region)::value;
    if (role == kRoleLoad) {
        for_each_segment([&](const Segment& sg, const int gstep) {
        FBF_SEGMENT_LOCALS
            // ============================ LOAD ==============================
            // fstage row q holds f at columns [xs, xs + FSW), border-mapped with
            // 4-byte cp.async (or one TMA bulk copy per row for the in-image span,
            // FBF_STAGE=bulk). Zero-border rows/columns outside the image are never
            // read: GEN treats them as zero.
            const float* src = p.src + (long long)sg.frame * p.src_frame_stride;
            // interior strips: the staged window [xs, xs + FSW) lies in the image and
            // rows are 16-byte aligned -> whole rows with 16-byte cp.async
            const bool vec = p.vec_ok && !p.use_tma && xs >= 0 && xs + FSW <= p.width;
            const int c0 = max(xs, 0), c1 = min(xs + FSW, p.width);  // in-image span
            const bool bulk = p.use_tma && c1 > c0;
            constexpr int LCOLS = (GW + 31) / 32;
            int lmx[LCOLS], loff[LCOLS];
            if (!vec) {
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
                if (g >= NFS) PSYNC(0, kBarFsEmpty + fb, kFsThreads);
                float* fs = fstage + fb * Q * FSW;
                const int a = a0 + s * Q;
                const int lo = max(a, ya - R), hi = min(a + Q, yb + R);
#ifdef FBF_SKIP_LOAD
                if (tid == 0) mbar_arrive(&fs_full[fb]);
                continue;
#endif
                // interior step (every row in the image, the window inside the row): one
                // tensor-map TMA of the whole Q x FSW tile. Rows the band's source window
                // lacks are outside the map (zero fill); they feed no stored output.
#ifndef FBF_NO_TMA2D
                if (p.use_tma2d && xs >= 0 && xs + FSW <= p.width && a >= 0 && a + Q <= p.height) {
                    if (tid == 0) {
                        mbar_expect_tx(&fs_full[fb], (unsigned)(sizeof(float) * Q * FSW));
                        tma_tile_g2s(fs, &tmap, xs, a - p.src_row0, sg.frame, &fs_full[fb]);
                        mbar_arrive(&fs_full[fb]);
                    }
                    continue;
                }
#endif
                if (vec) {
                    constexpr int NV = FSW / 4;  // float4 per staged row
                    constexpr int VITER = (Q * NV + 31) / 32;
#pragma unroll 1
                    for (int it = 0; it < VITER; ++it) {
                        const int i = it * 32 + tid;
                        if (i < Q * NV) {
                            const int q = i / NV, c = i - q * NV;
                            const int gy = a + q;
                            const int my = (gy >= lo && gy < hi) ? map_border(gy, p.height, p.border) : -1;
                            if (my >= 0)
                                cp_async16(fs + q * FSW + 4 * c, src + (long long)(my - p.src_row0) * p.src_pitch + xs + 4 * c);
                        }
                    }
                } else {
                    if (bulk) {
                        int nrows_src = 0;  // needed rows that read the image
                        for (int gy = lo; gy < hi; ++gy) nrows_src += map_border(gy, p.height, p.border) >= 0;
                        if (tid == 0 && nrows_src > 0)
                            mbar_expect_tx(&fs_full[fb], (unsigned)(sizeof(float) * (c1 - c0) * nrows_src));
                        __syncwarp();
                        if (tid < Q) {
                            const int gy = a + tid;
                            const int my = (gy >= lo && gy < hi) ? map_border(gy, p.height, p.border) : -1;
                            if (my >= 0)
                                tma_bulk_g2s(fs + tid * FSW + (c0 - xs),
                                             src + (long long)(my - p.src_row0) * p.src_pitch + c0,
                                             (unsigned)(sizeof(float) * (c1 - c0)), &fs_full[fb]);
                        }
                    }
#pragma unroll
                    for (int q = 0; q < Q; ++q) {
                        const int gy = a + q;
                        const int my = (gy >= lo && gy < hi) ? map_border(gy, p.height, p.border) : -1;
                        if (my < 0) continue;
                        const float* srow = src + (long long)(my - p.src_row0) * p.src_pitch;
#pragma unroll
                        for (int j = 0; j < LCOLS; ++j)
                            if (lmx[j] >= 0) cp_async4(fs + q * FSW + loff[j], srow + lmx[j]);
                    }
                }
                cp_async_mbar_arrive(&fs_full[fb]);
                __syncwarp();
                if (tid == 0) mbar_arrive(&fs_full[fb]);
            }
        });
    } else if (role == kRoleGen) {
        for_each_segment([&](const Segment& sg, const int gstep) {
        FBF_SEGMENT_LOCALS
            // ============================= GEN ==============================
            GenItem gi[GITER];
            gen_items(sg, gi);
            for (int t = 0; t < steps; ++t) {
                const int g = gstep + t;
                const int fb = g % NFS, gb = (g & (ngb - 1));
                PWAIT(0, &fs_full[fb], (unsigned)((g / NFS) & 1));
                if (g >= ngb) PSYNC(1, kBarGenEmpty + gb, gen_threads);
#ifndef FBF_SKIP_GEN
#ifdef FBF_DEV_LIGHT_W0  // dev: only the light warps on the lone-pair sub-partition work
                if (tid < 32)
#endif
                gen_step(sg, t, fb, gb, gi);
#endif
                // this warp's part of gen buffer gb written, fstage fb read
                named_arrive(kBarFsEmpty + fb, kFsThreads);
                named_arrive(kBarGenFull + gb, gen_threads);
            }
        });
    } else if (role == kRoleComb) {
        // duo: exchange slot s = xstep & 1 of the xstep-th output step; rank 1 writes the peer's
        // slot after the peer freed it (empty[s], arrived remotely), then arrives on the
        // peer's full[s]; rank 0 waits full[s], reads, and arrives on rank 1's empty[s]
        unsigned xpeer_slot = 0, xpeer_bar = 0;
        if (duo) {
            const unsigned peer = crank ^ 1u;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(xpeer_slot) : "r"(smem_u32(xslot)), "r"(peer));
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(xpeer_bar) : "r"(smem_u32(xbar)), "r"(peer));
        }
        constexpr unsigned XI = Q * (kTW / 2);  // pixel pairs per output step
        for_each_segment([&](const Segment& sg, const int gstep) {
        FBF_SEGMENT_LOCALS
            // ============================ COMB ==============================
            CombItem ci[CITER];
            comb_items(sg, ci);
            for (int t = 0; t < steps; ++t) {
                const int g = gstep + t;
                const int cb = (g & (ncb - 1));
                float2 fv[CITER];
                float4 nd[CITER];
                const unsigned slot = xstep & 1u, xpar = (xstep >> 1) & 1u;
                if (t >= s0) {
                    combine_load(sg, ci, fv, nd);
                    if (x_in) {  // the peer's (num, den) for these pixels
                        mbar_wait_cluster(&xbar[slot], xpar);
#pragma unroll
                        for (int it = 0; it < CITER; ++it) nd[it] = xslot[slot * XI + it * kCombThreads + tid];
                    }
                    if (x_out && xstep >= 2) mbar_wait_cluster(&xbar[2 + slot], xpar ^ 1u);  // the peer read slot
                }
                PSYNC(0, kBarColFull + cb, col_threads);
#ifndef FBF_SKIP_COMB
#ifdef FBF_DEV_LIGHT_W0
                if (tid < 32)
#endif
                if (t >= s0) combine_step(sg, cb, ci, fv, nd, xpeer_slot + slot * XI * 16u);
#endif
                if (duo && t >= s0) {
                    // rank 1: slot written -> peer's full[slot]; rank 0: slot read -> peer's empty[slot]
                    mbar_arrive_remote(xpeer_bar + 8u * (x_out ? slot : 2u + slot));
                    ++xstep;
                }
                named_arrive(kBarColEmpty + cb, col_threads);  // this warp is done with column buffer cb
            }
        });
    } else if (FMA && G::PAIR && role == kRoleRow) {
        for_each_segment([&](const Segment& sg, const int gstep) {
        FBF_SEGMENT_LOCALS
            // ============================= PAIR =============================
            // row pass of step t into the warp's own block, then the scatter column
            // pass of the same rows; the 2R column partial sums stay in registers
            if constexpr (FMA && G::PAIR) {
                const int pr = tid / 32;
                const int q = lane % Q, xc = lane / Q;
                float2* hbuf = ring + (size_t)pr * RROWS * RS;
                // per-buffer addresses, selected per step (no per-step address arithmetic)
                const float4* gin0 = reinterpret_cast<const float4*>(gen + ((size_t)pr * Q + q) * GS + xc * Q);
                const float4* gin1 = gin0 + (size_t)np * Q * GS / 2;
                float* oc0 = reinterpret_cast<float*>(colout + (size_t)pr * Q * kTW) + lane;
                float* oc1 = oc0 + (size_t)np * Q * kTW * 2;
                float2 st[2 * R];
#pragma unroll
                for (int i = 0; i < 2 * R; ++i) st[i] = make_float2(0.f, 0.f);  // new segment
                for (int t = 0; t < steps; ++t) {
                    const int g = gstep + t;
                    const int gb = (g & (ngb - 1)), cb = (g & (ncb - 1));
                    PSYNC(0, kBarGenFull + gb, gen_threads);
                    row_pass<R, Q>(gb ? gin1 : gin0, hbuf + (size_t)q * RS + xc * Q, p, kBarGenEmpty + gb, gen_threads);
                    __syncwarp();  // the step's row-pass block is complete
                    // column buffer cb must have been consumed by COMB even on warm-up steps:
                    // the arrival below completes a phase of col_full[cb]
                    if (g >= ncb) PSYNC(1, kBarColEmpty + cb, col_threads);
                    col_scatter<R, Q>(hbuf + lane, st, cb ? oc1 : oc0, t >= s0, p);
                    named_arrive(kBarColFull + cb, col_threads);
                }
            }
        });
    } else if (FMA && role == kRoleRow) {
        for_each_segment([&](const Segment& sg, const int gstep) {
        FBF_SEGMENT_LOCALS
            // ============================= ROW ==============================
            if constexpr (FMA && !G::PAIR) {
                const int pr = tid / 32;  // this warp's channel pair
                const int q = lane % Q, xc = lane / Q;
                static_assert(Q * (kTW / Q) == 32, "one warp covers a step of one pair");
                float2* myring = ring + (size_t)pr * RROWS * RS;
                const float4* gin0 = reinterpret_cast<const float4*>(gen + ((size_t)pr * Q + q) * GS + xc * Q);
                const float4* gin1 = gin0 + (size_t)np * Q * GS / 2;
                float2* hout0 = myring + (size_t)q * RS + xc * Q;
                for (int t = 0; t < steps; ++t) {
                    const int g = gstep + t;
                    const int gb = (g & (ngb - 1)), blk = g % RBP;
                    PSYNC(0, kBarGenFull + gb, gen_threads);
                    // ring block blk last held step g - RBP, read up to column pass g - RBP + RBN - 1
                    if constexpr (RING_NB) {
                        if (g >= 2) PSYNC(1, kBarRingEmpty + (g & 1), ring_threads);  // COL done with step g - 2
                    } else if (g >= RBP) {
                        PWAIT(1, &ring_empty[pr * RBP + blk], (unsigned)((g / RBP - 1) & 1));
                    }
                    row_pass<R, Q>(gb ? gin1 : gin0, hout0 + (size_t)blk * Q * RS, p, kBarGenEmpty + gb, gen_threads);
                    __syncwarp();  // ring block complete
                    if constexpr (RING_NB) named_arrive(kBarRingFull + (g & 1), ring_threads);
                    else if (lane == 0) mbar_arrive(&ring_full[pr * RBP + blk]);
                }
            }
        });
    } else if (FMA && role == kRoleCol) {
        for_each_segment([&](const Segment& sg, const int gstep) {
        FBF_SEGMENT_LOCALS
            // ============================= COL ==============================
            const int pr = tid / 32;
            const float2* myring = ring + (size_t)pr * RROWS * RS;
            if constexpr (!FMA || G::PAIR) {
            } else if constexpr (is_half(M)) {
                const int pr = tid / 64, h = (tid / 32) & 1;  // pair, output-row parity
                const float2* hring = ring + (size_t)pr * RROWS * RS;
                const float2* hin0 = hring + lane;
                const float2* hin1 = hin0 + (size_t)Q * RS;  // RBP == 2
                float* oc0 = reinterpret_cast<float*>(colout + (size_t)pr * Q * kTW) + lane;
                float* oc1 = oc0 + (size_t)np * Q * kTW * 2;
                float2 st[R];
#pragma unroll
                for (int i = 0; i < R; ++i) st[i] = make_float2(0.f, 0.f);  // new segment
                for (int t = 0; t < steps; ++t) {
                    const int g = gstep + t;
                    const int blk = g % RBP, cb = (g & (ncb - 1));
                    if constexpr (RING_NB) PSYNC(0, kBarRingFull + (g & 1), ring_threads);
                    else PWAIT(0, &ring_full[pr * RBP + blk], (unsigned)((g / RBP) & 1));
                    if (g >= ncb) PSYNC(1, kBarColEmpty + cb, col_threads);
                    float* oc = cb ? oc1 : oc0;
                    const float2* hin = blk ? hin1 : hin0;
                    if (h == 0) col_scatter_half<R, Q, 0>(hin, st, oc, t >= s0, p);
                    else col_scatter_half<R, Q, 1>(hin, st, oc, t >= s0, p);
                    if constexpr (RING_NB) named_arrive(kBarRingEmpty + (g & 1), ring_threads);  // COL done with step g
                    else if (__syncwarp(), lane == 0) mbar_arrive(&ring_empty[pr * RBP + blk]);
                    named_arrive(kBarColFull + cb, col_threads);
                }
            } else if constexpr (G::SCATTER) {
                const float2* hin0 = myring + lane;
                const float2* hin1 = hin0 + (size_t)Q * RS;  // RBP == 2
                float* oc0 = reinterpret_cast<float*>(colout + (size_t)pr * Q * kTW) + lane;
                float* oc1 = oc0 + (size_t)np * Q * kTW * 2;
                float2 st[2 * R];
#pragma unroll
                for (int i = 0; i < 2 * R; ++i) st[i] = make_float2(0.f, 0.f);  // new segment
                for (int t = 0; t < steps; ++t) {
                    const int g = gstep + t;
                    const int blk = g % RBP, cb = (g & (ncb - 1));
                    if constexpr (RING_NB) PSYNC(0, kBarRingFull + (g & 1), ring_threads);
                    else PWAIT(0, &ring_full[pr * RBP + blk], (unsigned)((g / RBP) & 1));
                    // column buffer cb must have been consumed by COMB even on warm-up steps:
                    // the arrival below completes a phase of col_full[cb]
                    if (g >= ncb) PSYNC(1, kBarColEmpty + cb, col_threads);
                    col_scatter<R, Q>(blk ? hin1 : hin0, st, cb ? oc1 : oc0, t >= s0, p);
                    if constexpr (RING_NB) named_arrive(kBarRingEmpty + (g & 1), ring_threads);  // COL done with step g
                    else if (__syncwarp(), lane == 0) mbar_arrive(&ring_empty[pr * RBP + blk]);
                    named_arrive(kBarColFull + cb, col_threads);
                }
            } else {
                for (int t = 0; t < steps; ++t) {
                    const int g = gstep + t;
                    const int blk = g % RBP, cb = (g & (ncb - 1));
                    const bool do_col = t >= s0;
                    if constexpr (RING_NB) PSYNC(0, kBarRingFull + (g & 1), ring_threads);
                    else PWAIT(0, &ring_full[pr * RBP + blk], (unsigned)((g / RBP) & 1));
                    float2 acc[Q];
                    if (do_col) col_pass<R, Q>(myring, blk, lane, p, acc);
                    // the oldest block of the window (step g - RB + 1) is free for row pass g - RB + 1 + RBP
                    if constexpr (RING_NB) named_arrive(kBarRingEmpty + (g & 1), ring_threads);  // COL done with step g
                    else if (__syncwarp(), lane == 0 && g >= RB - 1) mbar_arrive(&ring_empty[pr * RBP + (g - RB + 1) % RBP]);
                    // column buffer cb must have been consumed by COMB even on warm-up steps:
                    // the arrival below completes a phase of col_full[cb]
                    if (g >= ncb) PSYNC(1, kBarColEmpty + cb, col_threads);
                    if (do_col) {
                        float* oc = reinterpret_cast<float*>(colout + ((size_t)cb * np + pr) * Q * kTW) + lane;
#pragma unroll
                        for (int o = 0; o < Q; ++o) {  // planar: [channel][q][TW]
                            oc[o * kTW] = acc[o].x;
                            oc[(Q + o) * kTW] = acc[o].y;
                        }
                    }
                    named_arrive(kBarColFull + cb, col_threads);
                }
            }
        });
    }
    };  // run_roles
#undef FBF_SEGMENT_LOCALS
#ifdef FBF_DEV_PAIRONLY
    if (role != kRoleRow) role = kRoleIdle;
#endif
#ifndef FBF_NO_REGSPLIT
    if constexpr (M == kHalfWgMode) {
        // Half mode, 5 pairs, 24 warps (c4): the host places gen + combine in
        // warpgroups 0-1 (64 registers) and loader, ROW and COL-half warps in 2-5 (88):
        // at the uniform 80 the COL halves (R float2 partial sums) spill their loop
        // state around every step. 8 x 64 + 16 x 88 = 24 x 80. Its own instantiation:
        // a second, unsplit copy of the roles in the same function made ptxas spill
        // the COL loops of both copies.
        static_assert(FBF_WG_LO + 2 * FBF_WG_HI == 3 * 80, "8 warps at LO + 16 at HI must equal 24 warps at 80");
        if (threadIdx.x < 256) {
            asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(FBF_WG_LO));
            if (role != kRoleIdle) run_roles(std::false_type{});
        } else {
            asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(FBF_WG_HI));
            if (role != kRoleIdle) run_roles(std::true_type{});
        }
    } else if constexpr (M == kPairMode && NKR == 3) {
        // Register split between warpgroups (pair mode, 7 pairs, 16 warps): warpgroups
        // 0-1 (gen, combine) give up registers, 2-3 (loader + 7 pair warps) take them,
        // so the pair warps' row pass can keep loads in flight next to the 2r live
        // column partial sums. 8 x 96 + 8 x 160 = 16 x 128.
        if (blockDim.x == 512 && np == 7) {
            if (threadIdx.x < 256) {
                asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(FBF_REGSPLIT_LO));
                if (role != kRoleIdle) run_roles(std::false_type{});
            } else {
                asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(FBF_REGSPLIT_HI));
                run_roles(std::true_type{});
            }
        } else if (role != kRoleIdle) {
            run_roles(std::true_type{});
        }
    } else
#endif
    {
        if (role != kRoleIdle) run_roles(std::true_type{});
    }
    if (role == kRoleComb && p.fallbacks) {
        const unsigned w = __reduce_add_sync(0xffffffffu, n_fallbacks);
        if (lane == 0 && w) atomicAdd(p.fallbacks, (unsigned long long)w);
    }
    // duo: neither CTA exits while its peer may still write its exchange slots or
    // arrive on its barriers
    if (duo) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
#ifdef FBF_PHASES
    if (p.prof && lane == 0) {
        unsigned long long* pw = p.prof + 4 * (threadIdx.x / 32);
        atomicAdd(pw + 0, (unsigned long long)(clock64() - _pt0));
        atomicAdd(pw + 1, (unsigned long long)_pw[0]);
        atomicAdd(pw + 2, (unsigned long long)_pw[1]);
        atomicAdd(pw + 3, 1ull);
    }
#endif
}

template <int R, int Q, int NKR, int M>
cudaError_t launch_fused(const Params& p, const CUtensorMap& tmap, int grid, cudaStream_t stream) {
    using G = Geometry<R, Q, M>;
    // duo: both CTAs allocate the larger rank's layout plus the exchange region
    const int np_max = p.duo ? std::max(p.duo_chunk[0].n_pairs, p.duo_chunk[1].n_pairs) : p.n_pairs;
    const size_t smem = p.duo ? align128(G::smem_bytes(np_max, p.ngb, p.ncb)) + duo_xchg_bytes(Q)
                              : G::smem_bytes(p.n_pairs, p.ngb, p.ncb);
    // The dynamic shared-memory opt-in is a property of the function in the
    // CURRENT device's context: set it once per device (bit d of the mask), safe
    // against concurrent launches from the per-device host threads (a second
    // setter only repeats an idempotent call).
    static std::atomic<unsigned long long> configured{0};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(configured.load(std::memory_order_acquire) & bit)) {
        e = cudaFuncSetAttribute(fbf_fused_kernel<R, Q, NKR, M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kSmemLimit);
        if (e != cudaSuccess) return e;
        configured.fetch_or(bit, std::memory_order_acq_rel);
    }
    // programmatic stream serialization (host's choice, Params::pdl): the launch may
    // begin while the previous kernel on the stream finishes; the kernel waits for it
    // (griddepcontrol.wait) before touching global memory
    const bool pdl = p.pdl != 0;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block_threads(np_max, M));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    if (p.duo) {  // clusters of 2 CTAs (instead of PDL)
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
    }
    cfg.attrs = attr;
    cfg.numAttrs = (pdl || p.duo) ? 1 : 0;
    e = cudaLaunchKernelEx(&cfg, fbf_fused_kernel<R, Q, NKR, M>, p, tmap);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace fbf_dev
