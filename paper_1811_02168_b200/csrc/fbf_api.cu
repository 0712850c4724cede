// fbf_api.cu -- host side of the filtering path behind the C ABI (include/fbf.h).
//
// Mirrors fbf::fast_bilateral (/root/reference/proj/include/fourierbf/filter.hpp:43-46,
// src/filter.cpp:129-213): argument checks and error classes follow the
// reference (invalid_argument -> FBF_EINVAL, pixel range -> FBF_ERANGE), the
// numerical work runs in the fused sm_100a kernel (fbf_kernel.cuh).
//
// One context per CUDA device owns a stream, a cached device arena and a
// pinned counter block; calls on the same device serialise on its mutex, calls
// on different devices run concurrently. Multi-GPU entry points start one host
// thread per device: frames round-robin in contiguous blocks, or row bands with
// replicated radius-row halos. There is no collective: outputs are disjoint.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <atomic>
#include <chrono>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/fbf.h"
#include "fbf_cuda_util.h"
#include "fbf_internal.h"
#include "fbf_kernel.cuh"

namespace fbf_dev {
#include "fbf_kernel_extern.inc"

namespace {

using LaunchFn = cudaError_t (*)(const Params&, const CUtensorMap&, int, cudaStream_t);
// One step-height variant of a radius: launchers by NKR (number of k >= 1 terms
// in the launch) and the channel pairs that fit per CTA for each (gen buffers,
// column buffers) choice.
struct QEntry {
    LaunchFn launch[kMaxKR + 1] = {};
    int max_pairs[3][3] = {};  // [ngb][ncb], 1..2
    int duo_max_pairs[3][3] = {};  // the same with the duo exchange region appended
};
struct RadiusEntry {
    QEntry split8;          // split mode, Q = 8 (every radius)
    QEntry half8;           // half mode, Q = 8 (every radius, <= 7 pairs)
    QEntry half8wg;         // half mode with the warpgroup register split (5 pairs, NKR = 2 only)
    QEntry pair8, pair16;   // pair mode, r <= kQ16MaxRadius
};

template <int R, int Q, int M>
QEntry qentry() {
    using G = Geometry<R, Q, M>;
    QEntry e;
    e.launch[0] = &launch_fused<R, Q, 0, M>;
    e.launch[1] = &launch_fused<R, Q, 1, M>;
    e.launch[2] = &launch_fused<R, Q, 2, M>;
    e.launch[3] = &launch_fused<R, Q, 3, M>;
    if constexpr (!is_half(M)) e.launch[4] = &launch_fused<R, Q, 4, M>;
    for (int ngb = 1; ngb <= 2; ++ngb)
        for (int ncb = 1; ncb <= 2; ++ncb) {
            e.max_pairs[ngb][ncb] = is_half(M) ? std::min(kHalfMaxPairs, G::max_pairs(ngb, ncb))
                                                   : G::max_pairs(ngb, ncb);
            int d = e.max_pairs[ngb][ncb];
            while (d > 0 && align128(G::smem_bytes(d, ngb, ncb)) + duo_xchg_bytes(Q) > kSmemLimit) --d;
            e.duo_max_pairs[ngb][ncb] = d;
        }
    return e;
}

template <int R>
RadiusEntry entry() {
    RadiusEntry e;
#ifdef FBF_DEV_RADIUS  // dev builds with a single radius specialised (build.py --radius)
    if constexpr (R != FBF_DEV_RADIUS) return e;
#endif
    e.split8 = qentry<R, 8, kSplitMode>();
    e.half8 = qentry<R, 8, kHalfMode>();
    e.half8wg = e.half8;
    e.half8wg.launch[0] = e.half8wg.launch[1] = e.half8wg.launch[3] = nullptr;
    e.half8wg.launch[2] = &launch_fused<R, 8, 2, kHalfWgMode>;
    if constexpr (R <= kQ16MaxRadius) {
        e.pair8 = qentry<R, 8, kPairMode>();
        e.pair16 = qentry<R, 16, kPairMode>();
    }
    return e;
}

const RadiusEntry& radius_entry(int r) {
    static const RadiusEntry table[kMaxRadius + 1] = {
        RadiusEntry{}, entry<1>(),  entry<2>(),  entry<3>(),  entry<4>(),  entry<5>(),
        entry<6>(),  entry<7>(),  entry<8>(),  entry<9>(),  entry<10>(), entry<11>(),
        entry<12>(), entry<13>(), entry<14>(), entry<15>(), entry<16>(), entry<17>(),
        entry<18>(), entry<19>(), entry<20>(), entry<21>(), entry<22>(), entry<23>(),
        entry<24>(), entry<25>(), entry<26>(), entry<27>(), entry<28>(), entry<29>(),
        entry<30>(), entry<31>(), entry<32>()};
    return table[r];
}

// filter.cpp:19-23 on the device: flag any non-finite pixel or one outside [0, R]
__global__ void validate_kernel(const float* __restrict__ img, size_t n, float R, unsigned int* flag) {
    bool bad = false;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const float v = img[i];
        bad |= !(isfinite(v) && v >= 0.f && v <= R);
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1u);
}

// 8-bit I/O (imageio.cpp:53-101): bytes widen exactly to float; results are
// written like the CLI's write_clamped + write_pgm (fourierbf.cpp:71-76,
// imageio.cpp:83-89): clamp to [0, 255], round half away from zero
__global__ void u8_to_f32_kernel(const unsigned char* __restrict__ in, float* __restrict__ out, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        out[i] = (float)in[i];
}
__global__ void f32_to_u8_kernel(const float* __restrict__ in, unsigned char* __restrict__ out, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        out[i] = (unsigned char)roundf(fminf(255.f, fmaxf(0.f, in[i])));
}

}  // namespace
}  // namespace fbf_dev

namespace fbf_b200 {
namespace {

using fbf_dev::kTW;

int cuda_fail(cudaError_t e, const char* what) {
    return fail(FBF_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define FBF_CUDA(call, what)                                    \
    do {                                                        \
        cudaError_t e_ = (call);                                \
        if (e_ != cudaSuccess) return cuda_fail(e_, what);      \
    } while (0)

struct DeviceCtx {
    int device = 0;
    int num_sms = 0;
    cudaStream_t stream = nullptr;      // compute
    cudaStream_t stream_in = nullptr;   // host -> device copies
    cudaStream_t stream_out = nullptr;  // device -> host copies
    std::vector<cudaEvent_t> events;    // pipelining pool
    std::vector<cudaEvent_t> tevents;   // timing events (fbf_stage_timings)
    cudaMemPool_t pool = nullptr;       // stream-ordered scratch of the device-resident calls
    std::mutex mtx;
    void* arena = nullptr;  // cached device scratch
    size_t arena_bytes = 0;
    unsigned long long* d_counters = nullptr;  // [0] fallbacks, [1] range flag
    unsigned long long* h_counters = nullptr;  // pinned mirror

    int init(int dev) {
        device = dev;
        FBF_CUDA(cudaSetDevice(dev), "cudaSetDevice");
        FBF_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev), "attr");
        FBF_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
        FBF_CUDA(cudaStreamCreateWithFlags(&stream_in, cudaStreamNonBlocking), "cudaStreamCreate");
        FBF_CUDA(cudaStreamCreateWithFlags(&stream_out, cudaStreamNonBlocking), "cudaStreamCreate");
        FBF_CUDA(cudaMalloc(&d_counters, 2 * sizeof(unsigned long long)), "cudaMalloc counters");
        FBF_CUDA(cudaMallocHost(&h_counters, 2 * sizeof(unsigned long long)), "cudaMallocHost");
        // The device-resident entry points take their multi-chunk (num, den) scratch
        // from this pool in stream order (cudaMallocFromPoolAsync / cudaFreeAsync on
        // the caller's stream): calls on different streams never share scratch, and
        // nothing they enqueue touches the host path's arena. Freed blocks stay cached.
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        FBF_CUDA(cudaMemPoolCreate(&pool, &props), "cudaMemPoolCreate");
        unsigned long long keep = ~0ull;
        FBF_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep), "cudaMemPoolSetAttribute");
        return FBF_OK;
    }
    int timing_event(size_t i, cudaEvent_t* ev) {
        while (tevents.size() <= i) {
            cudaEvent_t e;
            FBF_CUDA(cudaEventCreate(&e), "cudaEventCreate");
            tevents.push_back(e);
        }
        *ev = tevents[i];
        return FBF_OK;
    }
    int event(size_t i, cudaEvent_t* ev) {
        while (events.size() <= i) {
            cudaEvent_t e;
            FBF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
            events.push_back(e);
        }
        *ev = events[i];
        return FBF_OK;
    }
    int reserve(size_t bytes) {
        if (bytes <= arena_bytes) return FBF_OK;
        if (arena) cudaFree(arena);
        arena = nullptr;
        arena_bytes = 0;
        const size_t want = bytes + bytes / 8;
        if (cudaMalloc(&arena, want) != cudaSuccess) {
            cudaGetLastError();
            return fail(FBF_ENOMEM, "device arena allocation of " + std::to_string(want) + " bytes failed");
        }
        arena_bytes = want;
        return FBF_OK;
    }
};

std::mutex g_ctx_mtx;
std::vector<std::unique_ptr<DeviceCtx>> g_ctx;
std::atomic<int> g_default_device{0};
std::atomic<unsigned long long> g_launches{0};

int get_ctx(int dev, DeviceCtx** out) {
    std::lock_guard<std::mutex> lock(g_ctx_mtx);
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return fail(FBF_ECUDA, "no CUDA device available (the fbf filter has no CPU fallback)");
    }
    if (dev < 0 || dev >= n) return fail(FBF_EINVAL, "device index out of range");
    if ((int)g_ctx.size() < n) g_ctx.resize(n);
    if (!g_ctx[dev]) {
        auto c = std::make_unique<DeviceCtx>();
        const int rc = c->init(dev);
        if (rc != FBF_OK) return rc;
        g_ctx[dev] = std::move(c);
    }
    *out = g_ctx[dev].get();
    return FBF_OK;
}

// ---- launch planning -------------------------------------------------------

struct Approx {
    int K = 0, T = 0, R = 0;
    double nu = 0.0;  // approx.frequency (filter.cpp:139); 0 = frequency_of(T)
    std::vector<double> c;
    // turns per intensity unit, nu / (2 pi), as the kernel's FP32 parameter
    float turns() const {
        const double from_T = 2.0 * 3.14159265358979323846 / (2.0 * T + 1.0);
        if (nu == 0.0 || nu == from_T) return (float)(1.0 / (2.0 * T + 1.0));
        return (float)(nu / (2.0 * 3.14159265358979323846));
    }
};

int check_args(int width, int height, double theta, int K, int T, int R, const double* coeffs,
               int border, int* radius) {
    // filter.cpp:132-134, kernels.cpp:106-107, image.hpp:21-22
    if (width <= 0 || height <= 0) return fail(FBF_EINVAL, "GrayImage: dimensions must be positive");
    if (!(theta > 0.0) || !std::isfinite(theta)) return fail(FBF_EINVAL, "spatial kernel: theta must be positive");
    if (K < 1 || T < 1 || R < 1 || !coeffs) return fail(FBF_EINVAL, "fast_bilateral: malformed approximation");
    if (border < 0 || border > 2) return fail(FBF_EINVAL, "unknown border policy");
    const int r = (int)std::ceil(3.0 * theta);
    if (r > fbf_dev::kMaxRadius)
        return fail(FBF_ECAPACITY, "spatial radius " + std::to_string(r) + " exceeds the kernel limit " +
                                       std::to_string(fbf_dev::kMaxRadius));
    *radius = r;
    return FBF_OK;
}

struct Chunk {
    int k_lo, n_k, n_pairs;
};

struct Plan {
    std::vector<Chunk> chunks;
    int q = 8, mode = 1, ngb = 2, ncb = 2;
    const fbf_dev::QEntry* ent = nullptr;
    const fbf_dev::QEntry* ent_wg = nullptr;  // half mode: the warpgroup-split variant (5 pairs)
};

// Split k = 0..K-1 into launches whose channel pairs fit in shared memory
// (k = 0 contributes one pair (f, 1), every k >= 1 two; at most kMaxKR terms
// k >= 1 per launch), balancing pair counts.
std::vector<Chunk> split_chunks(int K, int max_pairs) {
    std::vector<Chunk> out;
    if (max_pairs < 2) max_pairs = 2;  // always room for one k >= 1 term
    const int total = 2 * K - 1;
    const int n_chunks = (total + max_pairs - 1) / max_pairs;
    const int target = (total + n_chunks - 1) / n_chunks;
    int k = 0;
    while (k < K) {
        Chunk c{k, 0, 0};
        while (k < K) {
            const int add = k == 0 ? 1 : 2;
            const int nkr = c.n_k - (c.k_lo == 0 ? 1 : 0) + (k == 0 ? 0 : 1);
            if (c.n_k > 0 && (c.n_pairs + add > target || c.n_pairs + add > max_pairs || nkr > fbf_dev::kMaxKR))
                break;
            c.n_pairs += add;
            ++c.n_k;
            ++k;
        }
        out.push_back(c);
    }
    return out;
}

int env_int(const char* name) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : 0;
}

// FFMA2 warps per SM sub-partition (warp id mod 4) are what limits a CTA:
// the busiest sub-partition sets the pace, so a layout with w FFMA2 warps of
// equal work reaches at most w / (4 ceil(w / 4)) of the FMA peak.
double subpartition_balance(int warps) { return warps / (4.0 * ((warps + 3) / 4)); }

// One CTA per SM. Variant choice: fewest coefficient chunks first; then the
// warp organisation by measured rank: pair mode while its FFMA2 warps balance
// over the sub-partitions to >= 0.85 (c1: 7 pairs, 7/8), else half mode (up to 7
// pairs; c4: 0.60 vs 0.51 split), else split mode (c3: 9 pairs, 18 warps 9/10);
// then the preference list (Q, buffers). FBF_Q, FBF_MODE, FBF_NGB, FBF_NCB
// override (tuning).
// short_work: fewer than 64 output rows per CTA (small images, c0 512x512: 55): the
// launch is latency-bound and Q = 16 pair mode wins even with more chunks (c0:
// 24.7 us in two pair-mode launches vs 26.8 us in one split-mode launch)
Plan make_plan(int K, int r, bool short_work = false) {
    const auto& ent = fbf_dev::radius_entry(r);
    static const int fq = env_int("FBF_Q"), fngb = env_int("FBF_NGB"), fncb = env_int("FBF_NCB");
    static const int fmode = std::getenv("FBF_MODE") ? env_int("FBF_MODE") : -1;
    struct Pref {
        int q, mode, ngb, ncb;
    };
    constexpr int P = fbf_dev::kPairMode, S = fbf_dev::kSplitMode, H = fbf_dev::kHalfMode;
    static const Pref prefs[] = {{8, H, 2, 2}, {16, P, 2, 2}, {8, P, 2, 2}, {8, S, 2, 2}, {16, P, 2, 1},
                                 {8, H, 1, 1}, {8, P, 1, 1}, {8, S, 1, 1}, {16, P, 1, 1}};
    Plan best;
    double best_bal = -1.0;
    // overrides first; a radius without a matching variant takes the free choice
    for (int forced = 1; forced >= 0 && !best.ent; --forced) {
        for (const Pref& pf : prefs) {
            const fbf_dev::QEntry* qe = pf.mode == H   ? &ent.half8
                                        : pf.mode == S ? &ent.split8
                                        : pf.q == 16   ? &ent.pair16
                                                       : &ent.pair8;
            if (!qe->launch[0]) continue;
            if (forced && ((fq && fq != pf.q) || (fmode >= 0 && fmode != pf.mode) || (fngb && fngb != pf.ngb) ||
                           (fncb && fncb != pf.ncb)))
                continue;
            const int mp = qe->max_pairs[pf.ngb][pf.ncb];
            if (mp < 2) continue;
            auto chunks = split_chunks(K, mp);
            // half mode with 6-7 pairs runs 27-30 warps at 72 / 64 registers: from
            // r = 22 on the column-half warps' r partial sums spill heavily (measured,
            // 2048^2, split vs half: K = 4 (7 pairs) r 24 / 27 / 30: 0.59 / 0.56 / 0.56 vs
            // 0.54 / 0.48 / 0.42; K = 6 r 24 / 30: 0.54 / 0.47 vs 0.50 / 0.40; K = 9 r 30:
            // 0.45 vs 0.38; at 5 pairs half stays ahead: K = 5 r 27 / 30 0.49 / 0.50 vs
            // split 0.44 / 0.47; r 18 / 21, K = 4: half 0.47 / 0.51 vs split 0.44 / 0.50)
            if (fmode < 0 && pf.mode == H && r >= 22 &&
                std::any_of(chunks.begin(), chunks.end(), [](const Chunk& c) { return c.n_pairs >= 6; }))
                continue;
            double bal = 1.0;
            for (const Chunk& c : chunks) bal = std::min(bal, subpartition_balance((pf.mode == S ? 2 : 1) * c.n_pairs));
            // rank: 2 pair mode balanced >= 0.85, 1 half mode, 0 the rest (split, unbalanced pair)
            const double rank = pf.mode == P && bal >= 0.85 ? 2 : pf.mode == H ? 1 : 0;
            bal = rank + bal / 2;  // rank first, then balance
            bool better = best_bal < 0 || chunks.size() < best.chunks.size() ||
                          (chunks.size() == best.chunks.size() && bal > best_bal + 1e-9);
            if (short_work && fmode < 0 && best.ent) {
                const bool cand16 = pf.mode == P && pf.q == 16, best16 = best.mode == P && best.q == 16;
                if (cand16 != best16) better = cand16;
            }
            if (better) {
                best = Plan{std::move(chunks), pf.q, pf.mode, pf.ngb, pf.ncb, qe, pf.mode == H ? &ent.half8wg : nullptr};
                best_bal = bal;
            }
        }
    }
    return best;
}

// dev builds (FBF_PHASES) with FBF_PROF=1: per-warp-slot cycle counters
unsigned long long* g_prof = nullptr;
unsigned long long* dev_prof_buffer() {
#ifdef FBF_PHASES
    static const bool on = std::getenv("FBF_PROF") != nullptr;
    if (on && !g_prof && cudaMalloc(&g_prof, 128 * sizeof(unsigned long long)) == cudaSuccess)
        cudaMemset(g_prof, 0, 128 * sizeof(unsigned long long));
#endif
    return g_prof;
}

struct Job {
    const float* d_src;
    long long src_frame_stride;
    int src_row0, src_rows;
    float* d_dst;
    long long dst_frame_stride;
    int width, height, n_frames;
    int out_row0, out_rows;
};

// Half mode warp placement: sub-partition = warp id mod 4. The FFMA2 work is
// spread evenly (ROW warps weigh 2, each COL half 1), the light roles by their
// estimated issue load; within a sub-partition the FFMA2 warps take the highest
// warp ids (the issue arbiter serves higher ids first), unused slots idle.
// Returns true when it wrote the fixed warpgroup layout of the kHalfWgMode kernel.
bool half_mode_placement(int np, fbf_dev::Params& p) {
    using namespace fbf_dev;
    const int W = block_threads(np, kHalfMode) / 32, per = W / 4;
    // 5 pairs (c4): a fixed warpgroup layout for the kernel's register split -- gen and
    // combine in warpgroups 0-1 (64 registers), loader + ROW + COL halves in 2-5 (88).
    // FFMA2 weight per sub-partition (warp id mod 4; ROW 2, COL half 1): 5 5 5 5.
    static const bool no_split = std::getenv("FBF_HALF_SPLIT") && std::atoi(std::getenv("FBF_HALF_SPLIT")) == 0;
    if (np == 5 && W == 24 && !no_split) {
        constexpr unsigned char G = kRoleGen, M = kRoleComb, L = kRoleLoad, C = kRoleCol, R = kRoleRow;
        static const unsigned char layouts[3][24] = {
            {G, G, G, G, M, M, M, M, L, C, C, C, C, C, C, C, R, C, C, C, R, R, R, R},   // ROW warps highest
            {G, G, G, G, M, M, M, M, R, R, R, R, R, C, C, C, C, C, C, C, L, C, C, C},   // ROW warps lowest
            {G, G, G, G, M, M, M, M, L, C, C, C, R, R, R, R, C, C, C, C, R, C, C, C}};  // mixed
        static const int which = std::getenv("FBF_WG_PERM") ? std::atoi(std::getenv("FBF_WG_PERM")) % 3 : 0;
        const unsigned char* role = layouts[which];
        int next[6] = {0, 0, 0, 0, 0, 0};
        for (int w = 0; w < 32; ++w) {
            p.warp_role[w] = w < 24 ? role[w] : (unsigned char)kRoleIdle;
            p.warp_idx[w] = w < 24 ? (unsigned char)next[role[w]]++ : 0;
        }
        return true;
    }
    struct Item {
        int role, idx;
        double w;
        bool fma;
    };
    std::vector<Item> items;
    for (int i = 0; i < np; ++i) items.push_back({kRoleRow, i, 2.0, true});
    for (int i = 0; i < 2 * np; ++i) items.push_back({kRoleCol, i, 1.0, true});
    for (int i = 0; i < kGenWarps; ++i) items.push_back({kRoleGen, i, 0.6, false});
    for (int i = 0; i < kCombWarps; ++i) items.push_back({kRoleComb, i, 0.4, false});
    items.push_back({kRoleLoad, 0, 0.4, false});
    double load[4] = {0, 0, 0, 0};
    std::vector<Item> sub[4];
    for (const Item& it : items) {
        int best = -1;
        for (int s = 0; s < 4; ++s)
            if ((int)sub[s].size() < per && (best < 0 || load[s] < load[best] - 1e-9)) best = s;
        sub[best].push_back(it);
        load[best] += it.w;
    }
    for (int w = 0; w < 32; ++w) {
        p.warp_role[w] = kRoleIdle;
        p.warp_idx[w] = 0;
    }
    for (int s = 0; s < 4; ++s) {
        int lo = 0, hi = per - 1;  // slot k of sub-partition s is warp s + 4k
        for (const Item& it : sub[s]) {
            const int k = it.fma ? hi-- : lo++;
            p.warp_role[s + 4 * k] = (unsigned char)it.role;
            p.warp_idx[s + 4 * k] = (unsigned char)it.idx;
        }
    }
    return false;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (libfbf.so does
// not link libcuda: it must load on machines without a driver, and the filter
// then fails with FBF_ECUDA).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// The source of a job as a 3-D tensor (columns, rows present, frames) with a box of
// one f staging tile: FSW = the kernel's staged row width, Q rows, one frame.
int encode_source_map(const Job& job, int r, int q, CUtensorMap* map) {
    static EncodeTiledFn enc = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &qr) !=
                cudaSuccess || qr != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            fn = nullptr;
        }
        return (EncodeTiledFn)fn;
    }();
    if (!enc) return fail(FBF_ECUDA, "cuTensorMapEncodeTiled unavailable");
    const int gw = kTW + 2 * r, fsw = (gw + 3 + 3) / 4 * 4;  // Geometry::FSW
    cuuint64_t dims[3] = {(cuuint64_t)job.width, (cuuint64_t)job.src_rows, (cuuint64_t)job.n_frames};
    cuuint64_t strides[2] = {(cuuint64_t)job.width * sizeof(float),
                             (cuuint64_t)(job.n_frames > 1 ? job.src_frame_stride : (long long)job.width * job.src_rows) *
                                 sizeof(float)};
    cuuint32_t box[3] = {(cuuint32_t)fsw, (cuuint32_t)q, 1}, es[3] = {1, 1, 1};
    const CUresult rc = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(job.d_src), dims, strides, box,
                            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rc != CUDA_SUCCESS) return fail(FBF_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)rc));
    return FBF_OK;
}

// Runs every chunk launch for one job on `stream`. `scratch` must hold
// n_frames * out_rows * width float2 when K needs more than one chunk.
int run_job(DeviceCtx& ctx, const Job& job, double theta, const Approx& a, int border,
            float2* scratch, unsigned long long* d_fallbacks, cudaStream_t stream,
            unsigned int* d_bad = nullptr) {
    const int r = (int)std::ceil(3.0 * theta);
    const long long units = (long long)job.n_frames * ((job.width + kTW - 1) / kTW) * job.out_rows;
    const Plan plan = make_plan(a.K, r, units < 64LL * ctx.num_sms);
    if (!plan.ent) return fail(FBF_ECAPACITY, "no kernel variant fits the shared memory for this radius");
    if (plan.chunks.size() > 1 && !scratch) return fail(FBF_EINVAL, "internal: scratch required");
    static const bool log_plan = std::getenv("FBF_PLAN_LOG") != nullptr;  // dev: print the launch plan
    if (log_plan) {
        std::string line = "fbf plan: K=" + std::to_string(a.K) + " r=" + std::to_string(r) + " mode=" +
                           std::to_string(plan.mode) + " Q=" + std::to_string(plan.q) + " ngb=" +
                           std::to_string(plan.ngb) + " ncb=" + std::to_string(plan.ncb) + " chunks:";
        for (const Chunk& c : plan.chunks) line += " " + std::to_string(c.n_pairs);
        std::fprintf(stderr, "%s units=%lld\n", line.c_str(), units);
    }

    fbf_dev::Params p{};
    CUtensorMap tmap{};
    p.src = job.d_src;
    p.src_frame_stride = job.src_frame_stride;
    p.src_pitch = job.width;
    p.src_row0 = job.src_row0;
    p.src_rows = job.src_rows;
    p.dst = job.d_dst;
    p.dst_frame_stride = job.dst_frame_stride;
    p.dst_pitch = job.width;
    p.acc = plan.chunks.size() > 1 ? scratch : nullptr;
    p.acc_frame_stride = (long long)job.out_rows * job.width;
    p.fallbacks = d_fallbacks;
    p.bad_pixels = d_bad;
    p.range_max = (float)a.R;
    p.width = job.width;
    p.height = job.height;
    p.n_frames = job.n_frames;
    p.border = border;
    p.out_row0 = job.out_row0;
    p.out_rows = job.out_rows;
    p.n_strips = (job.width + kTW - 1) / kTW;
    p.total_units = (long long)job.n_frames * p.n_strips * job.out_rows;
    // kernels.cpp:105-118 taps, kept by |d|
    for (int j = 0; j <= r; ++j)
        p.taps[j] = p.taps_col[j] = (float)std::exp(-((double)j * j) / (2.0 * theta * theta));
    // interior row spans go through the TMA bulk-copy engine when rows are 16-byte aligned
    // Interior f rows: element cp.async by default (measured fastest on B200:
    // profiles/r01_stage_modes.txt); FBF_STAGE=bulk routes them through the TMA
    // bulk-copy engine (needs 16-byte aligned rows).
    // FBF_STAGE (dev): "tma" (default) interior tiles by 2-D tensor-map TMA, "elem"
    // element / 16-byte cp.async only, "bulk" 1-D bulk copies per row
    static const int stage_mode = [] {
        const char* e = std::getenv("FBF_STAGE");
        if (e && std::strcmp(e, "bulk") == 0) return 1;
        if (e && std::strcmp(e, "elem") == 0) return 2;
        return 0;
    }();
    const bool aligned = job.width % 4 == 0 && ((uintptr_t)job.d_src & 15) == 0 &&
                         (job.n_frames == 1 || job.src_frame_stride % 4 == 0);
    p.use_tma = aligned && stage_mode == 1 ? 1 : 0;
    p.vec_ok = aligned ? 1 : 0;
    p.use_tma2d = 0;
    if (aligned && stage_mode == 0) {
        const int rc = encode_source_map(job, r, plan.q, &tmap);
        if (rc != FBF_OK) return rc;
        p.use_tma2d = 1;
    }
    // persistent grid: CTAs per SM x SMs, but keep segments at least a few steps long
    p.ngb = plan.ngb;
    p.prof = dev_prof_buffer();
    p.ncb = plan.ncb;
    const long long min_seg = 4 * plan.q;
    const long long want = (p.total_units + min_seg - 1) / min_seg;
    const int grid = (int)std::max(1LL, std::min<long long>((long long)ctx.num_sms, want));
    // Whole columns (frame, strip) round-robin over the CTAs first: neighbouring strips
    // stream the same rows at the same time, so the halo columns they share are read
    // from DRAM once (c4: 3.24 -> 1.26 GB read per launch for a 1.07 GB input, time
    // unchanged); then a contiguous split of the rest. FBF_ORDER=contig (dev): the
    // plain contiguous split.
    static const bool contig = [] {
        const char* e = std::getenv("FBF_ORDER");
        return e && std::strcmp(e, "contig") == 0;
    }();
    p.col_rounds = contig ? 0 : (int)(((long long)job.n_frames * p.n_strips) / grid);
    // Programmatic dependent launch for short launches (< 512 output rows per CTA: the
    // next grid's launch and prologue overlap this one's drain): c0 24.8 -> 24.0 us,
    // one c3 frame 0.499 -> 0.513. Long launches lose with it (c4 0.701 -> 0.693, c2
    // 0.599 -> 0.591: the dependent grid's CTAs land on SMs in drain order, not launch
    // order). FBF_PDL=0 / 1 (dev) forces it off / on.
    static const int pdl_env = [] {
        const char* v = std::getenv("FBF_PDL");
        return v ? std::atoi(v) : -1;
    }();
    // (r02e: threshold 1024 -> 512 rows per CTA. Back-to-back c1 launches, 885 rows per CTA,
    // lose with it: 0.572 without, 0.548-0.557 with; a 2048 x 2048 image at r = 9, K = 4
    // 0.427 vs 0.364. c0 (55 rows) 24.3 vs 25.7 us and one c3 frame (438 rows) 0.519 vs
    // 0.508 keep it.)
    p.pdl = pdl_env >= 0 ? pdl_env : (p.total_units < 512LL * grid ? 1 : 0);
    p.inv_period = a.turns();

    // Duo launch for two-chunk plans (c2: K = 9, 9 + 8 pairs): clusters of 2 CTAs, each
    // work share filtered by both ranks at once, rank 1's (num, den) partials handed to
    // rank 0 per step through distributed shared memory -- one launch, no HBM scratch,
    // the same bits as the two scratch launches. FBF_DUO=0 (dev) keeps the scratch path, 1 forces the duo.
    static const int duo_env = std::getenv("FBF_DUO") ? std::atoi(std::getenv("FBF_DUO")) : -1;  // dev: 0 off, 1 on at any radius
    const bool duo_off = duo_env == 0;
    auto nkr_of = [](const Chunk& c) { return c.n_k - (c.k_lo == 0 ? 1 : 0); };
    // Small radii keep the two scratch launches (2048 x 2048, K = 9: r = 6 / 9 / 12 0.283 / 0.392 /
    // 0.521 with the scratch vs 0.268 / 0.377 / 0.480 as a duo; r = 15 0.550 vs 0.554): a duo step
    // ends with the cross-CTA handoff, which short steps do not amortise.
    if (!duo_off && plan.chunks.size() == 2 && plan.mode != fbf_dev::kHalfMode && ctx.num_sms >= 2 && (r >= 14 || duo_env == 1) &&
        nkr_of(plan.chunks[0]) == nkr_of(plan.chunks[1]) &&
        std::max(plan.chunks[0].n_pairs, plan.chunks[1].n_pairs) <= plan.ent->duo_max_pairs[plan.ngb][plan.ncb]) {
        const int clusters = (int)std::max(1LL, std::min<long long>((long long)ctx.num_sms / 2, (want + 1) / 2));
        p.duo = 1;
        p.pdl = 0;
        p.acc = nullptr;
        p.col_rounds = contig ? 0 : (int)(((long long)job.n_frames * p.n_strips) / clusters);
        for (int rk = 0; rk < 2; ++rk) {
            const Chunk& c = plan.chunks[rk == 0 ? 1 : 0];  // rank 0: the last chunk (writes the output)
            auto& d = p.duo_chunk[rk];
            d.k_lo = c.k_lo;
            d.n_pairs = c.n_pairs;
            d.k_first = std::max(c.k_lo, 1);
            for (int kk = 0; kk < c.n_k; ++kk) d.coeff[kk] = (float)a.c[c.k_lo + kk];
        }
        p.n_pairs = std::max(plan.chunks[0].n_pairs, plan.chunks[1].n_pairs);
        const cudaError_t e = plan.ent->launch[nkr_of(plan.chunks[0])](p, tmap, 2 * clusters, stream);
        if (e != cudaSuccess) return cuda_fail(e, "fbf_fused_kernel duo launch");
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return FBF_OK;
    }

    for (size_t ci = 0; ci < plan.chunks.size(); ++ci) {
        const Chunk& c = plan.chunks[ci];
        const int zk = c.k_lo == 0 ? 1 : 0;
        const int nkr = c.n_k - zk;
        p.k_lo = c.k_lo;
        p.n_pairs = c.n_pairs;
        p.first_chunk = ci == 0;
        p.last_chunk = ci + 1 == plan.chunks.size();
        for (int kk = 0; kk < c.n_k; ++kk) p.coeff[kk] = (float)a.c[c.k_lo + kk];
        p.k_first = std::max(c.k_lo, 1);
        const bool wg = plan.mode == fbf_dev::kHalfMode && half_mode_placement(c.n_pairs, p);
        const fbf_dev::QEntry* qe = wg ? plan.ent_wg : plan.ent;  // every radius has the split variant
        const cudaError_t e = qe->launch[nkr](p, tmap, grid, stream);
        if (e != cudaSuccess) return cuda_fail(e, "fbf_fused_kernel launch");
        g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    return FBF_OK;
}

size_t scratch_bytes(const Approx& a, double theta, size_t pixels) {
    const int r = (int)std::ceil(3.0 * theta);
    // either plan (short_work or not) may run, so size for both
    const bool chunked = make_plan(a.K, r).chunks.size() > 1 || make_plan(a.K, r, true).chunks.size() > 1;
    return chunked ? pixels * sizeof(float2) : 0;
}

size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }

void source_window(int height, int out_row0, int out_rows, int r, int border, int* row0, int* rows);

// Host buffers of a call: float32, or 8-bit (PGM payloads) widened / rounded on the device.
struct HostIO {
    const void* in;
    void* out;
    bool in_u8 = false, out_u8 = false;
    size_t in_elem() const { return in_u8 ? 1 : sizeof(float); }
    size_t out_elem() const { return out_u8 ? 1 : sizeof(float); }
};

// What one host-buffer call on one device covers: n_frames whole frames, or
// (n_frames == 1) output rows [out_row0, out_row0 + out_rows) of a
// width x height image whose rows [src_row0, src_row0 + src_rows) are at io.in
// (a row band plus the halo the border mapping reaches; the whole image for a
// single-image call). io.out receives the output rows only.
struct Window {
    int n_frames = 1;
    int src_row0 = 0, src_rows = 0;
    int out_row0 = 0, out_rows = 0;
};

// Stage busy times of a call (fbf_stage_timings), from timing events.
struct StageClock {
    double h2d = 0, kernel = 0, d2h = 0;
};

// Host-buffer path on one device. The work is cut into pieces (row sub-bands
// of the window, or groups of frames) and pipelined over three streams: H2D of
// piece i+1 and D2H of piece i-1 overlap the kernel of piece i; intensity
// validation is fused into the kernel. A sub-band's kernel reads the whole
// device-resident window, so halos need no extra copies: it waits for the copy
// of the last source piece its border-mapped rows reach. Results are identical
// to one launch over the window. On any failure after the first enqueue the
// three streams are drained before returning, so no copy into or out of the
// caller's buffers is still in flight (out is then undefined).
int filter_on_device(int dev, const HostIO& io, const Window& wd, int width, int height, double theta,
                     const Approx& a, int border, long long* fallbacks, StageClock* clock) {
    DeviceCtx* ctx = nullptr;
    int rc = get_ctx(dev, &ctx);
    if (rc != FBF_OK) return rc;
    std::lock_guard<std::mutex> lock(ctx->mtx);
    DeviceGuard dguard;
    FBF_CUDA(cudaSetDevice(dev), "cudaSetDevice");
    const bool bands = wd.n_frames == 1;
    const size_t fp = (size_t)width * height;
    const size_t in_px = bands ? (size_t)wd.src_rows * width : (size_t)wd.n_frames * fp;
    const size_t out_px = bands ? (size_t)wd.out_rows * width : (size_t)wd.n_frames * fp;
    const size_t in_bytes = align_up(in_px * sizeof(float)), out_bytes = align_up(out_px * sizeof(float));
    const size_t scr = align_up(scratch_bytes(a, theta, out_px));
    const size_t in8 = io.in_u8 ? align_up(in_px) : 0, out8 = io.out_u8 ? align_up(out_px) : 0;
    rc = ctx->reserve(in_bytes + out_bytes + scr + in8 + out8);
    if (rc != FBF_OK) return rc;
    float* d_in = (float*)ctx->arena;
    float* d_out = (float*)((char*)ctx->arena + in_bytes);
    float2* d_scr = scr ? (float2*)((char*)ctx->arena + in_bytes + out_bytes) : nullptr;
    unsigned char* d_in8 = (unsigned char*)ctx->arena + in_bytes + out_bytes + scr;
    unsigned char* d_out8 = d_in8 + in8;
    const int cvt_grid = ctx->num_sms * 8;
    cudaStream_t sc = ctx->stream, si = ctx->stream_in, so = ctx->stream_out;
    struct Drain {  // error paths: nothing of this call may still be running afterwards
        cudaStream_t s[3];
        bool armed = true;
        ~Drain() {
            if (!armed) return;
            for (cudaStream_t x : s) cudaStreamSynchronize(x);
            cudaGetLastError();
        }
    } drain{{si, sc, so}};
    unsigned int* d_flag = (unsigned int*)(ctx->d_counters + 1);
    const int r = (int)std::ceil(3.0 * theta);
    FBF_CUDA(cudaMemsetAsync(ctx->d_counters, 0, 2 * sizeof(unsigned long long), si), "memset");

    // bands: one piece per ~4 MiB crossing PCIe (in + out), at most 8 -- more pieces
    // overlap more transfer with compute but each band kernel pays 2r warm-up rows
    // (c1: float32 8 pieces 0.56 ms vs 4 pieces 0.59; 8-bit 2 pieces 0.37 ms vs 8: 0.46)
    const long long io_bytes = (long long)in_px * (long long)io.in_elem() + (long long)out_px * io.out_elem();
    int pieces = bands ? (int)std::min<long long>(8, std::max<long long>(1, io_bytes / (4 << 20)))
                       : std::min(wd.n_frames, 16);
    // very large images: the first piece's H2D and the last piece's kernel + D2H are not
    // overlapped, so keep pieces near 64 MiB of traffic, up to 32 (c4, 1 GiB in + 1 GiB out:
    // 8 / 16 / 32 / 64 pieces 28.7 / 26.5 / 25.4 / 26.7 ms per call; c2, 64 MiB each way,
    // stays at 8: 3.29 ms vs 3.52 / 4.25 at 16 / 32)
    if (bands && io_bytes > (512LL << 20)) pieces = (int)std::min<long long>(32, io_bytes / (64LL << 20));
    if (bands) pieces = std::max(1, std::min(pieces, wd.out_rows / std::max(64, 4 * r)));
    static const int forced_pieces = env_int("FBF_PIECES");  // tuning override
    if (forced_pieces > 0) pieces = std::max(1, std::min(forced_pieces, bands ? wd.out_rows : wd.n_frames));
    // piece i: output rows [lo[i], lo[i+1]) (global rows) or frames [lo[i], lo[i+1]);
    // its input copy covers source rows [sb[i], sb[i+1]) (or the same frames)
    std::vector<int> lo(pieces + 1), sb(pieces + 1);
    for (int i = 0; i <= pieces; ++i) {
        lo[i] = bands ? wd.out_row0 + (int)((long long)wd.out_rows * i / pieces)
                      : (int)((long long)wd.n_frames * i / pieces);
        sb[i] = bands ? std::clamp(lo[i], wd.src_row0, wd.src_row0 + wd.src_rows) : lo[i];
    }
    if (bands) {
        sb[0] = wd.src_row0;
        sb[pieces] = wd.src_row0 + wd.src_rows;
    }
    const size_t unit = bands ? (size_t)width : fp;  // floats per row / per frame
    const long long in_base = bands ? wd.src_row0 : 0, out_base = bands ? wd.out_row0 : 0;
    cudaEvent_t ev;
    // timing events per piece: [h2d0, h2d1, k0, k1, d2h0, d2h1]
    auto tmark = [&](size_t piece, int which, cudaStream_t st) -> int {
        if (!clock) return FBF_OK;
        cudaEvent_t e;
        int rc2 = ctx->timing_event(6 * piece + which, &e);
        if (rc2 != FBF_OK) return rc2;
        FBF_CUDA(cudaEventRecord(e, st), "event");
        return FBF_OK;
    };
    for (int i = 0; i < pieces; ++i) {
        const size_t off = (size_t)(sb[i] - in_base) * unit, n = (size_t)(sb[i + 1] - sb[i]) * unit;
        if ((rc = tmark(i, 0, si)) != FBF_OK) return rc;
        if (n > 0) {
            if (io.in_u8) {
                FBF_CUDA(cudaMemcpyAsync(d_in8 + off, (const unsigned char*)io.in + off, n, cudaMemcpyHostToDevice,
                                         si), "H2D");
                fbf_dev::u8_to_f32_kernel<<<cvt_grid, 256, 0, si>>>(d_in8 + off, d_in + off, n);
                FBF_CUDA(cudaGetLastError(), "u8 widen launch");
                g_launches += 1;
            } else {
                FBF_CUDA(cudaMemcpyAsync(d_in + off, (const float*)io.in + off, n * sizeof(float),
                                         cudaMemcpyHostToDevice, si), "H2D");
            }
        }
        if ((rc = tmark(i, 1, si)) != FBF_OK) return rc;
        if ((rc = ctx->event(2 * i, &ev)) != FBF_OK) return rc;
        FBF_CUDA(cudaEventRecord(ev, si), "event");
    }
    for (int i = 0; i < pieces; ++i) {
        int need = i;  // last input piece this piece's window reaches
        if (bands) {
            int s0 = 0, sn = 0;
            source_window(height, lo[i], lo[i + 1] - lo[i], r, border, &s0, &sn);
            need = 0;
            while (need + 1 < pieces && sb[need + 1] < s0 + sn) ++need;
        }
        if ((rc = ctx->event(2 * need, &ev)) != FBF_OK) return rc;
        FBF_CUDA(cudaStreamWaitEvent(sc, ev, 0), "wait");
        Job job = bands ? Job{d_in, (long long)fp, wd.src_row0, wd.src_rows, d_out + (size_t)(lo[i] - out_base) * width,
                              (long long)fp, width, height, 1, lo[i], lo[i + 1] - lo[i]}
                        : Job{d_in + (size_t)lo[i] * fp, (long long)fp, 0, height, d_out + (size_t)lo[i] * fp,
                              (long long)fp, width, height, lo[i + 1] - lo[i], 0, height};
        const size_t ooff = (size_t)(lo[i] - out_base) * unit, on = (size_t)(lo[i + 1] - lo[i]) * unit;
        float2* sp = d_scr ? d_scr + ooff : nullptr;
        if ((rc = tmark(i, 2, sc)) != FBF_OK) return rc;
        // intensity validation runs inside the kernel (every pixel is combined once)
        rc = run_job(*ctx, job, theta, a, border, sp, ctx->d_counters, sc, d_flag);
        if (rc != FBF_OK) return rc;
        if (io.out_u8) {
            fbf_dev::f32_to_u8_kernel<<<cvt_grid, 256, 0, sc>>>(d_out + ooff, d_out8 + ooff, on);
            FBF_CUDA(cudaGetLastError(), "u8 round launch");
            g_launches += 1;
        }
        if ((rc = tmark(i, 3, sc)) != FBF_OK) return rc;
        if ((rc = ctx->event(2 * i + 1, &ev)) != FBF_OK) return rc;
        FBF_CUDA(cudaEventRecord(ev, sc), "event");
        FBF_CUDA(cudaStreamWaitEvent(so, ev, 0), "wait");
        if ((rc = tmark(i, 4, so)) != FBF_OK) return rc;
        if (io.out_u8)
            FBF_CUDA(cudaMemcpyAsync((unsigned char*)io.out + ooff, d_out8 + ooff, on, cudaMemcpyDeviceToHost, so),
                     "D2H");
        else
            FBF_CUDA(cudaMemcpyAsync((float*)io.out + ooff, d_out + ooff, on * sizeof(float), cudaMemcpyDeviceToHost,
                                     so), "D2H");
        if ((rc = tmark(i, 5, so)) != FBF_OK) return rc;
    }
    FBF_CUDA(cudaMemcpyAsync(ctx->h_counters, ctx->d_counters, 2 * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, so), "D2H counters");
    FBF_CUDA(cudaStreamSynchronize(so), "filter");
    drain.armed = false;
    if (clock) {
        for (int i = 0; i < pieces; ++i) {
            float ms[3] = {0, 0, 0};
            for (int k = 0; k < 3; ++k)
                FBF_CUDA(cudaEventElapsedTime(&ms[k], ctx->tevents[6 * i + 2 * k], ctx->tevents[6 * i + 2 * k + 1]),
                         "timing");
            clock->h2d += 1e-3 * ms[0];
            clock->kernel += 1e-3 * ms[1];
            clock->d2h += 1e-3 * ms[2];
        }
    }
    if (ctx->h_counters[1]) return fail(FBF_ERANGE, "filter: pixel intensity outside [0, R]");
    if (fallbacks) *fallbacks += (long long)ctx->h_counters[0];
    return FBF_OK;
}

int make_approx(int K, int T, int R, const double* coeffs, Approx& a, double frequency = 0.0) {
    a.K = K;
    a.T = T;
    a.R = R;
    if (!std::isfinite(frequency)) return fail(FBF_EINVAL, "fast_bilateral: non-finite frequency");
    a.nu = frequency;
    a.c.assign(coeffs, coeffs + K);
    for (double v : a.c)
        if (!std::isfinite(v)) return fail(FBF_EINVAL, "fast_bilateral: non-finite coefficient");
    return FBF_OK;
}

int resolve_gpus(int n_gpus, int* out) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return fail(FBF_ECUDA, "no CUDA device available (the fbf filter has no CPU fallback)");
    }
    *out = n_gpus <= 0 ? n : std::min(n_gpus, n);
    return FBF_OK;
}

// Runs fn(g) on one host thread per device and returns the first failure.
template <typename Fn>
int per_device(int G, Fn&& fn) {
    std::vector<int> rcs(G, FBF_OK);
    std::vector<std::string> msgs(G);
    std::vector<std::thread> th;
    for (int g = 0; g < G; ++g)
        th.emplace_back([&, g] {
            rcs[g] = fn(g);
            if (rcs[g] != FBF_OK) msgs[g] = fbf_last_error();
        });
    for (auto& t : th) t.join();
    for (int g = 0; g < G; ++g)
        if (rcs[g] != FBF_OK) return fail(rcs[g], msgs[g]);
    return FBF_OK;
}

void source_window(int height, int out_row0, int out_rows, int r, int border, int* row0, int* rows) {
    int lo = std::max(0, out_row0 - r), hi = std::min(height, out_row0 + out_rows + r);
    // halo rows outside the image reach back in through the border mapping
    auto widen = [&](int y) {
        if (y >= 0 && y < height) return;
        const int m = fbf_dev::map_border(y, height, border);
        if (m < 0) return;
        lo = std::min(lo, m);
        hi = std::max(hi, m + 1);
    };
    for (int y = out_row0 - r; y < out_row0; ++y) widen(y);
    for (int y = out_row0 + out_rows; y < out_row0 + out_rows + r; ++y) widen(y);
    *row0 = lo;
    *rows = hi - lo;
}

// Device-resident job on the caller's stream; multi-chunk scratch from the
// context's stream-ordered pool (allocated and freed on `st`).
int run_device_job(int device, const Job& job, double theta, const Approx& a, int border,
                   unsigned long long* d_fallbacks, cudaStream_t st) {
    DeviceCtx* ctx = nullptr;
    int rc = get_ctx(device, &ctx);
    if (rc != FBF_OK) return rc;
    DeviceGuard dguard;
    FBF_CUDA(cudaSetDevice(device), "cudaSetDevice");
    const size_t scr = scratch_bytes(a, theta, (size_t)job.n_frames * job.out_rows * job.width);
    float2* d_scr = nullptr;
    if (scr) {
        const cudaError_t e = cudaMallocFromPoolAsync((void**)&d_scr, scr, ctx->pool, st);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(e == cudaErrorMemoryAllocation ? FBF_ENOMEM : FBF_ECUDA,
                        std::string("scratch allocation: ") + cudaGetErrorString(e));
        }
    }
    rc = run_job(*ctx, job, theta, a, border, d_scr, d_fallbacks, st);
    if (d_scr) cudaFreeAsync(d_scr, st);
    return rc;
}

int band_of(int height, int G, int g, int* y0, int* y1) {
    *y0 = (int)((long long)height * g / G);
    *y1 = (int)((long long)height * (g + 1) / G);
    return *y1 - *y0;
}

}  // namespace

int device_context(int device, void** stream, std::mutex** mtx) {
    DeviceCtx* ctx = nullptr;
    const int rc = get_ctx(device, &ctx);
    if (rc != FBF_OK) return rc;
    *stream = ctx->stream;
    *mtx = &ctx->mtx;
    return FBF_OK;
}

void count_launch(unsigned long long n) { g_launches += n; }

}  // namespace fbf_b200

using namespace fbf_b200;

extern "C" {

int fbf_set_device(int device) {
    if (device < 0 || device >= fbf_device_count()) return fail(FBF_EINVAL, "device index out of range");
    g_default_device.store(device);
    return FBF_OK;
}

int fbf_get_device(void) { return g_default_device.load(); }

unsigned long long fbf_kernel_launches(void) { return g_launches.load(); }

// dev: read and reset the FBF_PHASES per-warp-slot counters (128 values); -1 if absent
int fbf_dev_prof(unsigned long long* out) {
    if (!fbf_b200::g_prof) return -1;
    cudaDeviceSynchronize();
    cudaMemcpy(out, fbf_b200::g_prof, 128 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaMemset(fbf_b200::g_prof, 0, 128 * sizeof(unsigned long long));
    return 0;
}

int fbf_host_alloc(size_t bytes, void** ptr) {
    // page-locked, portable across devices: the copy engines reach ~55 GB/s per
    // direction from these (measured against ~29 GB/s H2D from some other
    // pinned allocators, tools/microbench/h2d_probe.cu)
    *ptr = nullptr;
    if (bytes == 0) return fail(FBF_EINVAL, "host_alloc: zero bytes");
    const cudaError_t e = cudaHostAlloc(ptr, bytes, cudaHostAllocPortable);
    if (e != cudaSuccess) {
        *ptr = nullptr;
        return fail(e == cudaErrorMemoryAllocation ? FBF_ENOMEM : FBF_ECUDA,
                    std::string("cudaHostAlloc: ") + cudaGetErrorString(e));
    }
    return FBF_OK;
}

int fbf_host_free(void* ptr) {
    if (ptr) FBF_CUDA(cudaFreeHost(ptr), "cudaFreeHost");
    return FBF_OK;
}

int fbf_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int fbf_validate_f32_device(const float* d_img, size_t n, int R, int device, void* stream) {
    DeviceCtx* ctx = nullptr;
    int rc = get_ctx(device, &ctx);
    if (rc != FBF_OK) return rc;
    std::lock_guard<std::mutex> lock(ctx->mtx);
    DeviceGuard dguard;
    FBF_CUDA(cudaSetDevice(device), "cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;  // NULL = the legacy default stream
    FBF_CUDA(cudaMemsetAsync(ctx->d_counters + 1, 0, sizeof(unsigned long long), st), "memset");
    fbf_dev::validate_kernel<<<ctx->num_sms * 4, 256, 0, st>>>(d_img, n, (float)R,
                                                              (unsigned int*)(ctx->d_counters + 1));
    FBF_CUDA(cudaGetLastError(), "validate launch");
    FBF_CUDA(cudaMemcpyAsync(ctx->h_counters + 1, ctx->d_counters + 1, sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, st), "D2H");
    FBF_CUDA(cudaStreamSynchronize(st), "validate");
    if (ctx->h_counters[1]) return fail(FBF_ERANGE, "filter: pixel intensity outside [0, R]");
    return FBF_OK;
}

int fbf_fast_bilateral_ex(const float* img, int width, int height, double theta, int K, int T, int R,
                          double frequency, const double* coeffs, int border, float* out, long long* fallbacks,
                          fbf_stage_timings* timings) {
    const auto t0 = std::chrono::steady_clock::now();
    int r = 0;
    int rc = check_args(width, height, theta, K, T, R, coeffs, border, &r);
    if (rc != FBF_OK) return rc;
    if (!img || !out) return fail(FBF_EINVAL, "fast_bilateral: null image buffer");
    Approx a;
    rc = make_approx(K, T, R, coeffs, a, frequency);
    if (rc != FBF_OK) return rc;
    StageClock clock;
    Window wd{1, 0, height, 0, height};
    rc = filter_on_device(g_default_device.load(), HostIO{img, out}, wd, width, height, theta, a, border, fallbacks,
                          timings ? &clock : nullptr);
    if (rc != FBF_OK) return rc;
    if (timings) {  // accumulated like StageTimings (filter.cpp:151-211)
        timings->convolution_seconds += clock.kernel;
        timings->h2d_seconds += clock.h2d;
        timings->d2h_seconds += clock.d2h;
        timings->wall_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    clear_error();
    return FBF_OK;
}

int fbf_fast_bilateral_f32(const float* img, int width, int height, double theta, int K, int T, int R,
                           const double* coeffs, int border, float* out, long long* fallbacks) {
    return fbf_fast_bilateral_ex(img, width, height, theta, K, T, R, 0.0, coeffs, border, out, fallbacks, nullptr);
}

int fbf_fast_bilateral_f32_device(const float* d_img, int width, int height, double theta, int K, int T,
                                  int R, const double* coeffs, int border, float* d_out,
                                  unsigned long long* d_fallbacks, int device, void* stream) {
    return fbf_fast_bilateral_band_f32_device(d_img, 0, height, width, height, 0, height, theta, K, T, R,
                                              coeffs, border, d_out, d_fallbacks, device, stream);
}

int fbf_fast_bilateral_band_f32_device(const float* d_src, int src_row0, int src_rows, int width, int height,
                                       int out_row0, int out_rows, double theta, int K, int T, int R,
                                       const double* coeffs, int border, float* d_dst,
                                       unsigned long long* d_fallbacks, int device, void* stream) {
    int r = 0;
    int rc = check_args(width, height, theta, K, T, R, coeffs, border, &r);
    if (rc != FBF_OK) return rc;
    if (out_row0 < 0 || out_rows <= 0 || out_row0 + out_rows > height)
        return fail(FBF_EINVAL, "band: output rows outside the image");
    int need0 = 0, need_rows = 0;
    source_window(height, out_row0, out_rows, r, border, &need0, &need_rows);
    if (src_row0 > need0 || src_row0 + src_rows < need0 + need_rows)
        return fail(FBF_EINVAL, "band: source rows do not cover the halo");
    Approx a;
    rc = make_approx(K, T, R, coeffs, a);
    if (rc != FBF_OK) return rc;
    Job job{d_src, 0, src_row0, src_rows, d_dst, 0, width, height, 1, out_row0, out_rows};
    rc = run_device_job(device, job, theta, a, border, d_fallbacks, (cudaStream_t)stream);
    if (rc == FBF_OK) clear_error();
    return rc;
}

int fbf_fast_bilateral_batch_f32_device(const float* d_img, int n_frames, int width, int height, double theta, int K,
                                        int T, int R, const double* coeffs, int border, float* d_out,
                                        unsigned long long* d_fallbacks, int device, void* stream) {
    int r = 0;
    int rc = check_args(width, height, theta, K, T, R, coeffs, border, &r);
    if (rc != FBF_OK) return rc;
    if (n_frames <= 0) return fail(FBF_EINVAL, "batch: n_frames must be positive");
    Approx a;
    rc = make_approx(K, T, R, coeffs, a);
    if (rc != FBF_OK) return rc;
    const size_t fp = (size_t)width * height;
    // one launch over all frames: CTAs take contiguous (frame, strip, row) shares
    Job job{d_img, (long long)fp, 0, height, d_out, (long long)fp, width, height, n_frames, 0, height};
    rc = run_device_job(device, job, theta, a, border, d_fallbacks, (cudaStream_t)stream);
    if (rc == FBF_OK) clear_error();
    return rc;
}

int fbf_band_source_rows(int height, int out_row0, int out_rows, double theta, int border, int* row0,
                         int* rows) {
    if (!(theta > 0.0) || height <= 0 || out_rows <= 0 || out_row0 < 0 || out_row0 + out_rows > height)
        return fail(FBF_EINVAL, "band: invalid arguments");
    source_window(height, out_row0, out_rows, (int)std::ceil(3.0 * theta), border, row0, rows);
    return FBF_OK;
}

int fbf_fast_bilateral_batch_f32(const float* img, int n_frames, int width, int height, double theta, int K,
                                 int T, int R, const double* coeffs, int border, float* out,
                                 long long* fallbacks, int n_gpus) {
    int r = 0;
    int rc = check_args(width, height, theta, K, T, R, coeffs, border, &r);
    if (rc != FBF_OK) return rc;
    if (n_frames <= 0) return fail(FBF_EINVAL, "batch: n_frames must be positive");
    Approx a;
    rc = make_approx(K, T, R, coeffs, a);
    if (rc != FBF_OK) return rc;
    int G = 0;
    rc = resolve_gpus(n_gpus, &G);
    if (rc != FBF_OK) return rc;
    G = std::min(G, n_frames);
    const size_t fp = (size_t)width * height;
    std::vector<long long> fb(G, 0);
    rc = per_device(G, [&](int g) {
        const int f0 = (int)((long long)n_frames * g / G), f1 = (int)((long long)n_frames * (g + 1) / G);
        // one device: the process's default device (fbf_set_device), e.g. its local rank
        const int dev = G == 1 ? g_default_device.load() : g;
        Window wd{f1 - f0, 0, height, 0, height};
        return filter_on_device(dev, HostIO{img + f0 * fp, out + f0 * fp}, wd, width, height, theta, a, border,
                                &fb[g], nullptr);
    });
    if (rc != FBF_OK) return rc;
    if (fallbacks)
        for (long long v : fb) *fallbacks += v;
    clear_error();
    return FBF_OK;
}

int fbf_fast_bilateral_bands_f32(const float* img, int width, int height, double theta, int K, int T, int R,
                                 const double* coeffs, int border, float* out, long long* fallbacks,
                                 int n_gpus) {
    int r = 0;
    int rc = check_args(width, height, theta, K, T, R, coeffs, border, &r);
    if (rc != FBF_OK) return rc;
    Approx a;
    rc = make_approx(K, T, R, coeffs, a);
    if (rc != FBF_OK) return rc;
    int G = 0;
    rc = resolve_gpus(n_gpus, &G);
    if (rc != FBF_OK) return rc;
    G = std::max(1, std::min(G, height));
    std::vector<long long> fb(G, 0);
    // one host thread per device; each device pipelines its band + halo window
    // (H2D / kernel / D2H in sub-bands, like the single-image call)
    rc = per_device(G, [&](int g) -> int {
        int y0 = 0, y1 = 0;
        band_of(height, G, g, &y0, &y1);
        int s0 = 0, sn = 0;
        source_window(height, y0, y1 - y0, r, border, &s0, &sn);
        const int dev = G == 1 ? g_default_device.load() : g;
        Window wd{1, s0, sn, y0, y1 - y0};
        return filter_on_device(dev, HostIO{img + (size_t)s0 * width, out + (size_t)y0 * width}, wd, width, height,
                                theta, a, border, &fb[g], nullptr);
    });
    if (rc != FBF_OK) return rc;
    if (fallbacks)
        for (long long v : fb) *fallbacks += v;
    clear_error();
    return FBF_OK;
}

int fbf_fast_bilateral_band_f32(const float* src, int src_row0, int src_rows, int width, int height, int out_row0,
                                int out_rows, double theta, int K, int T, int R, const double* coeffs, int border,
                                float* out, long long* fallbacks) {
    int r = 0;
    int rc = check_args(width, height, theta, K, T, R, coeffs, border, &r);
    if (rc != FBF_OK) return rc;
    if (!src || !out) return fail(FBF_EINVAL, "fast_bilateral_band: null buffer");
    if (out_row0 < 0 || out_rows <= 0 || out_row0 + out_rows > height)
        return fail(FBF_EINVAL, "fast_bilateral_band: output rows outside the image");
    int s0 = 0, sn = 0;
    source_window(height, out_row0, out_rows, r, border, &s0, &sn);
    if (src_row0 < 0 || src_rows <= 0 || src_row0 + src_rows > height || src_row0 > s0 || src_row0 + src_rows < s0 + sn)
        return fail(FBF_EINVAL, "fast_bilateral_band: source rows do not cover the band's halo window");
    Approx a;
    rc = make_approx(K, T, R, coeffs, a);
    if (rc != FBF_OK) return rc;
    long long fb = 0;
    Window wd{1, src_row0, src_rows, out_row0, out_rows};
    rc = filter_on_device(g_default_device.load(), HostIO{src, out}, wd, width, height, theta, a, border, &fb, nullptr);
    if (rc != FBF_OK) return rc;
    if (fallbacks) *fallbacks += fb;
    clear_error();
    return FBF_OK;
}

int fbf_fast_bilateral_u8(const unsigned char* img, int width, int height, double theta, int K, int T, int R,
                          const double* coeffs, int border, unsigned char* out_u8, float* out_f32,
                          long long* fallbacks) {
    int r = 0;
    int rc = check_args(width, height, theta, K, T, R, coeffs, border, &r);
    if (rc != FBF_OK) return rc;
    if (!out_u8 && !out_f32) return fail(FBF_EINVAL, "fast_bilateral_u8: no output buffer");
    if (out_u8 && out_f32) return fail(FBF_EINVAL, "fast_bilateral_u8: give one output buffer");
    Approx a;
    rc = make_approx(K, T, R, coeffs, a);
    if (rc != FBF_OK) return rc;
    HostIO io{img, out_u8 ? (void*)out_u8 : (void*)out_f32, true, out_u8 != nullptr};
    Window wd{1, 0, height, 0, height};
    rc = filter_on_device(g_default_device.load(), io, wd, width, height, theta, a, border, fallbacks, nullptr);
    if (rc == FBF_OK) clear_error();
    return rc;
}

int fbf_filter(const float* img, int height, int width, double theta, double sigma, double eps_or_K,
               float* out) {
    // run_filter (tools/fourierbf.cpp:236-270) with the CLI defaults: Gaussian
    // kernel, R = 255, symmetric border
    const int R = 255;
    const bool is_K = eps_or_K >= 1.0 && std::floor(eps_or_K) == eps_or_K;
    std::vector<double> c(2 * R + 1);
    int K = 0, T = 0;
    double err = 0.0;
    // period scans on the GPU (same K, T, c as the host scan: fbf_scan.cu)
    int rc = fbf_select_params_gpu(FBF_KERNEL_GAUSSIAN, sigma, R, is_K ? 0.0 : eps_or_K, is_K ? (int)eps_or_K : 0,
                                   0, 0, g_default_device.load(), &K, &T, c.data(), (int)c.size(), &err);
    if (rc != FBF_OK) return rc;
    return fbf_fast_bilateral_f32(img, width, height, theta, K, T, R, c.data(), FBF_BORDER_SYMMETRIC, out,
                                  nullptr);
}

}  // extern "C"
