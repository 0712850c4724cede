// fbf_scan.cu -- the period scan of the host optimiser on the GPU.
//
// Replaces the inner loop of scan_period_errors / min_error_over_period
// (/root/reference/proj/src/approx.cpp:119-144) as called by
// optimize_parameters (approx.cpp:179-240) and the CLI's select_parameters
// (tools/fourierbf.cpp:185-234): E(K, T) = ||A c - b||^2 of the least-squares
// fit of the sampled range kernel b[2R+1] by the cosine design matrix A(K, T)
// (approx.cpp:61-103), for every T in 1..t_max and a batch of orders K.
//
// One CTA per (K, T) problem, FP64 throughout. A (m x K, column-major) lives
// in shared memory; the factorisation is the one of fbf_params.cpp (Householder
// QR with column pivoting on the largest remaining column norm, rank cut at
// 1e-10 |R_00|, minimum-norm solution on the rank-deficient branch), with the
// column norms and reflections parallel over rows (warp per column) and the
// small triangular / Cholesky solves on one thread. E is then evaluated on the
// regenerated original A, as approx.cpp:101 does.
//
// The tree reductions round differently from the host's sequential sums, so
// these errors agree with the host scan to ~1e-15 relative near the minimum
// (~1e-6 where A is ill-conditioned, far above it), not bit for bit. The host
// therefore re-evaluates, with its own routine, every T whose GPU error lies
// within a relative 1e-4 of the GPU minimum and takes the argmin of
// those exact values (strict '<', smaller T on ties): the selected (K, T) and
// its coefficients are exactly the host scan's (fbf_params.cpp).
#include <cuda_runtime.h>

#include <cmath>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/fbf.h"
#include "fbf_cuda_util.h"
#include "fbf_internal.h"

namespace fbf_dev {

constexpr int kScanThreads = 256;
constexpr int kScanWarps = kScanThreads / 32;
constexpr double kRankTol = 1e-10;  // approx.cpp:15

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Shared layout (doubles): A[m * Kc] | qb[m] | colv[Kc] (norms / dots) | u[Kc] | h[Kc] |
// S[Kc * Kc] | M[Kc * Kc] | rhs[Kc] | z[Kc] | red[kScanWarps]; perm[Kc] ints after.
__global__ void __launch_bounds__(kScanThreads) period_scan_kernel(const double* __restrict__ b, int R, int K_lo,
                                                                   int t_max, int Kc, double* __restrict__ errors) {
    extern __shared__ double sm[];
    const int m = 2 * R + 1;
    const int prob = blockIdx.x;
    const int K = K_lo + prob / t_max;
    const int T = 1 + prob % t_max;
    double* A = sm;
    double* qb = A + (size_t)m * Kc;
    double* colv = qb + m;
    double* u = colv + Kc;
    double* hv = u + Kc;
    double* S = hv + Kc;
    double* M = S + Kc * Kc;
    double* rhs = M + Kc * Kc;
    double* z = rhs + Kc;
    double* red = z + Kc;
    int* perm = reinterpret_cast<int*>(red + kScanWarps);
    __shared__ int s_rank, s_pivot;
    __shared__ double s_best, s_vj, s_vnorm2, s_alpha;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double nu = 2.0 * 3.14159265358979323846 / (2.0 * T + 1.0);  // approx.cpp:17-19

    // design matrix (approx.cpp:61-86): column j = cos(j nu t) by the Chebyshev recurrence
    for (int i = tid; i < m; i += kScanThreads) {
        const double c1 = cos(nu * (double)(i - R));
        A[i] = 1.0;
        if (K > 1) A[(size_t)m + i] = c1;
        for (int j = 2; j < K; ++j)
            A[(size_t)j * m + i] = 2.0 * c1 * A[(size_t)(j - 1) * m + i] - A[(size_t)(j - 2) * m + i];
        qb[i] = b[i];
    }
    for (int j = tid; j < K; j += kScanThreads) perm[j] = j;
    __syncthreads();

    const int steps = min(m, K);
    for (int j = 0; j < steps; ++j) {
        // remaining column norms over rows >= j, one warp per column
        for (int k = j + warp; k < K; k += kScanWarps) {
            const double* ck = A + (size_t)k * m;
            double s = 0.0;
            for (int i = j + lane; i < m; i += 32) s += ck[i] * ck[i];
            s = warp_sum(s);
            if (lane == 0) colv[k] = s;
        }
        __syncthreads();
        if (tid == 0) {  // first maximum (fbf_params.cpp: strict '>' over ascending k)
            int p = j;
            double best = -1.0;
            for (int k = j; k < K; ++k)
                if (colv[k] > best) {
                    best = colv[k];
                    p = k;
                }
            s_pivot = p;
            s_best = best;
            if (p != j) {
                const int t = perm[j];
                perm[j] = perm[p];
                perm[p] = t;
            }
        }
        __syncthreads();
        const int p = s_pivot;
        if (p != j)
            for (int i = tid; i < m; i += kScanThreads) {
                const double t = A[(size_t)j * m + i];
                A[(size_t)j * m + i] = A[(size_t)p * m + i];
                A[(size_t)p * m + i] = t;
            }
        __syncthreads();
        double* cj = A + (size_t)j * m;
        const double norm = sqrt(s_best);
        if (norm == 0.0) continue;  // uniform: every thread sees the same s_best
        if (warp == 0) {
            const double alpha = cj[j] > 0 ? -norm : norm;
            const double vj = cj[j] - alpha;
            double s = 0.0;
            for (int i = j + 1 + lane; i < m; i += 32) s += cj[i] * cj[i];
            s = warp_sum(s);
            if (lane == 0) {
                s_alpha = alpha;
                s_vj = vj;
                s_vnorm2 = vj * vj + s;
            }
        }
        __syncthreads();
        const double vj = s_vj, vnorm2 = s_vnorm2;
        if (vnorm2 != 0.0) {
            // reflect columns k > j and qb (index K), one warp per vector
            for (int k = j + 1 + warp; k <= K; k += kScanWarps) {
                double* x = k < K ? A + (size_t)k * m : qb;
                double s = 0.0;
                for (int i = j + 1 + lane; i < m; i += 32) s += cj[i] * x[i];
                s = warp_sum(s) + vj * x[j];
                const double f = 2.0 * s / vnorm2;
                for (int i = j + 1 + lane; i < m; i += 32) x[i] -= f * cj[i];
                __syncwarp();
                if (lane == 0) x[j] -= f * vj;
            }
        }
        __syncthreads();
        if (tid == 0) cj[j] = s_alpha;
        __syncthreads();
    }

    // rank, R11^{-1} g and the minimum-norm branch (fbf_params.cpp), one thread
    if (tid == 0) {
        auto Rij = [&](int i, int j) { return A[(size_t)j * m + i]; };
        const double maxpivot = fabs(A[0]);
        int rank = 0;
        for (int j = 0; j < steps; ++j)
            if (fabs(Rij(j, j)) > kRankTol * maxpivot) ++rank;
        for (int j = 0; j < K; ++j) u[j] = 0.0;
        if (rank > 0) {
            for (int i = rank - 1; i >= 0; --i) {
                double s = qb[i];
                for (int k = i + 1; k < rank; ++k) s -= Rij(i, k) * hv[k];
                hv[i] = s / Rij(i, i);
            }
            if (rank == K) {
                for (int i = 0; i < K; ++i) u[i] = hv[i];
            } else {
                const int q = K - rank;
                for (int c2 = 0; c2 < q; ++c2)
                    for (int i = rank - 1; i >= 0; --i) {
                        double s = Rij(i, rank + c2);
                        for (int k = i + 1; k < rank; ++k) s -= Rij(i, k) * S[k * q + c2];
                        S[i * q + c2] = s / Rij(i, i);
                    }
                for (int a = 0; a < q; ++a) {
                    rhs[a] = 0.0;
                    for (int bq = 0; bq < q; ++bq) {
                        double s = a == bq ? 1.0 : 0.0;
                        for (int i = 0; i < rank; ++i) s += S[i * q + a] * S[i * q + bq];
                        M[a * q + bq] = s;
                    }
                    for (int i = 0; i < rank; ++i) rhs[a] += S[i * q + a] * hv[i];
                }
                for (int a = 0; a < q; ++a)
                    for (int bq = 0; bq <= a; ++bq) {
                        double s = M[a * q + bq];
                        for (int k = 0; k < bq; ++k) s -= M[a * q + k] * M[bq * q + k];
                        M[a * q + bq] = a == bq ? sqrt(s) : s / M[bq * q + bq];
                    }
                for (int a = 0; a < q; ++a) {
                    double s = rhs[a];
                    for (int k = 0; k < a; ++k) s -= M[a * q + k] * z[k];
                    z[a] = s / M[a * q + a];
                }
                for (int a = q - 1; a >= 0; --a) {
                    double s = z[a];
                    for (int k = a + 1; k < q; ++k) s -= M[k * q + a] * z[k];
                    z[a] = s / M[a * q + a];
                }
                for (int i = 0; i < rank; ++i) {
                    double s = hv[i];
                    for (int a = 0; a < q; ++a) s -= S[i * q + a] * z[a];
                    u[i] = s;
                }
                for (int a = 0; a < q; ++a) u[rank + a] = z[a];
            }
        }
        // c[perm[j]] = u[j], kept in colv
        for (int j = 0; j < K; ++j) colv[perm[j]] = u[j];
        s_rank = rank;
    }
    __syncthreads();

    // E = ||A c - b||^2 on the regenerated original matrix (approx.cpp:101)
    double e = 0.0;
    for (int i = tid; i < m; i += kScanThreads) {
        const double c1 = cos(nu * (double)(i - R));
        double tkm2 = 1.0, tkm1 = c1;
        double s = colv[0];
        if (K > 1) s += c1 * colv[1];
        for (int j = 2; j < K; ++j) {
            const double tk = 2.0 * c1 * tkm1 - tkm2;
            s += tk * colv[j];
            tkm2 = tkm1;
            tkm1 = tk;
        }
        const double d = s - b[i];
        e += d * d;
    }
    e = warp_sum(e);
    if (lane == 0) red[warp] = e;
    __syncthreads();
    if (tid == 0) {
        double s = 0.0;
        for (int w = 0; w < kScanWarps; ++w) s += red[w];
        errors[prob] = s;
    }
}

size_t scan_smem_bytes(int m, int Kc) {
    return sizeof(double) * ((size_t)m * Kc + m + 6 * (size_t)Kc + 2 * (size_t)Kc * Kc + kScanWarps) +
           sizeof(int) * (size_t)Kc;
}

}  // namespace fbf_dev

namespace fbf_b200 {

int gpu_scan_max_order(int R) {
    const int m = 2 * R + 1;
    int k = 1;
    while (k < m && fbf_dev::scan_smem_bytes(m, k + 1) <= 200 * 1024) ++k;
    return k;
}

int gpu_scan_errors(const double* samples, int R, int K_lo, int nK, int t_max, int device, double* errors) {
    if (R < 1 || K_lo < 1 || nK < 1 || t_max < 1 || K_lo + nK - 1 > 2 * R + 1)
        return fail(FBF_EINVAL, "gpu period scan: invalid (R, K, t_max)");
    const int Kc = K_lo + nK - 1;
    if (Kc > gpu_scan_max_order(R))
        return fail(FBF_ECAPACITY, "gpu period scan: K = " + std::to_string(Kc) +
                                       " exceeds the shared-memory design matrix (max " +
                                       std::to_string(gpu_scan_max_order(R)) + ")");
    void* stream_v = nullptr;
    std::mutex* mtx = nullptr;
    int rc = device_context(device, &stream_v, &mtx);
    if (rc != FBF_OK) return rc;
    std::lock_guard<std::mutex> lock(*mtx);
    cudaStream_t st = (cudaStream_t)stream_v;
    const int m = 2 * R + 1;
    const size_t n = (size_t)nK * t_max;
    double *d_b = nullptr, *d_e = nullptr;
    auto cleanup = [&] {
        if (d_b) cudaFree(d_b);
        if (d_e) cudaFree(d_e);
    };
    auto cu = [&](cudaError_t e, const char* what) {
        if (e == cudaSuccess) return FBF_OK;
        cleanup();
        return fail(FBF_ECUDA, std::string("gpu period scan: ") + what + ": " + cudaGetErrorString(e));
    };
    DeviceGuard dguard;
    if ((rc = cu(cudaSetDevice(device), "cudaSetDevice")) != FBF_OK) return rc;
    if ((rc = cu(cudaMalloc(&d_b, sizeof(double) * m), "cudaMalloc")) != FBF_OK) return rc;
    if ((rc = cu(cudaMalloc(&d_e, sizeof(double) * n), "cudaMalloc")) != FBF_OK) return rc;
    if ((rc = cu(cudaMemcpyAsync(d_b, samples, sizeof(double) * m, cudaMemcpyHostToDevice, st), "H2D")) != FBF_OK)
        return rc;
    const size_t smem = fbf_dev::scan_smem_bytes(m, Kc);
    if ((rc = cu(cudaFuncSetAttribute(fbf_dev::period_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem),
                 "smem attribute")) != FBF_OK)
        return rc;
    fbf_dev::period_scan_kernel<<<(unsigned)n, fbf_dev::kScanThreads, smem, st>>>(d_b, R, K_lo, t_max, Kc, d_e);
    if ((rc = cu(cudaGetLastError(), "launch")) != FBF_OK) return rc;
    count_launch();
    if ((rc = cu(cudaMemcpyAsync(errors, d_e, sizeof(double) * n, cudaMemcpyDeviceToHost, st), "D2H")) != FBF_OK)
        return rc;
    if ((rc = cu(cudaStreamSynchronize(st), "sync")) != FBF_OK) return rc;
    cleanup();
    return FBF_OK;
}

}  // namespace fbf_b200
