// fbf_params.cpp -- host-side parameter selection (range-kernel sampling and
// the least-squares optimiser of (K, T, c)), restated without Eigen.
//
// Follows /root/reference/proj/src/kernels.cpp:19-32,78-118 and
// src/approx.cpp:17-19,61-240, and the CLI's select_parameters
// (tools/fourierbf.cpp:185-234). The reference solves each least-squares
// problem with Eigen's CompleteOrthogonalDecomposition (rank threshold 1e-10);
// Eigen is not available here, so this file implements the same factorisation
// family directly: Householder QR with column pivoting, a rank cut at
// 1e-10 * |R_00|, and the minimum-norm solution on the rank-deficient branch.
// Pinned against the reference's frozen values in tests/test_params.py.
#include <cmath>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <numbers>
#include <string>
#include <thread>
#include <vector>

#include "../../include/fbf.h"
#include "fbf_internal.h"

namespace fbf_b200 {

namespace {

thread_local std::string g_last_error;

constexpr double kRankTolerance = 1e-10;  // approx.cpp:15

// approx.cpp:61-86 -- column-major m x K, Chebyshev recurrence on cos(nu t).
bool design_matrix(int K, int T, int R, std::vector<double>& A) {
    if (K < 1 || T < 1 || R < 1 || K > 2 * R + 1) return false;
    const int m = 2 * R + 1;
    const double nu = fbf_frequency_of(T);
    A.assign(static_cast<size_t>(m) * K, 0.0);
    for (int i = 0; i < m; ++i) {
        const int t = i - R;
        A[i] = 1.0;
        if (K > 1) {
            const double c1 = std::cos(nu * t);
            A[static_cast<size_t>(m) + i] = c1;
            for (int j = 2; j < K; ++j)
                A[static_cast<size_t>(j) * m + i] =
                    2.0 * c1 * A[static_cast<size_t>(j - 1) * m + i] -
                    A[static_cast<size_t>(j - 2) * m + i];
        }
    }
    return true;
}

// approx.cpp:88-103 -- min-norm least squares of the m x n column-major A.
// Returns false on non-finite input (the reference throws runtime_error).
bool fit_coefficients(const std::vector<double>& A0, int m, int n, const double* b0,
                      std::vector<double>& c, double& err) {
    for (double v : A0)
        if (!std::isfinite(v)) return false;
    for (int i = 0; i < m; ++i)
        if (!std::isfinite(b0[i])) return false;

    std::vector<double> A(A0);
    std::vector<double> qb(b0, b0 + m);
    std::vector<int> perm(n);
    for (int j = 0; j < n; ++j) perm[j] = j;
    auto col = [&](int j) { return A.data() + static_cast<size_t>(j) * m; };

    // Householder QR with column pivoting (largest remaining column norm).
    const int steps = std::min(m, n);
    for (int j = 0; j < steps; ++j) {
        int p = j;
        double best = -1.0;
        for (int k = j; k < n; ++k) {
            double s = 0.0;
            const double* ck = col(k);
            for (int i = j; i < m; ++i) s += ck[i] * ck[i];
            if (s > best) {
                best = s;
                p = k;
            }
        }
        if (p != j) {
            std::swap_ranges(col(j), col(j) + m, col(p));
            std::swap(perm[j], perm[p]);
        }
        double* cj = col(j);
        const double norm = std::sqrt(best);
        if (norm == 0.0) continue;
        const double alpha = cj[j] > 0 ? -norm : norm;
        // v = x - alpha e1, stored in place below the diagonal (v_j kept apart)
        const double vj = cj[j] - alpha;
        double vnorm2 = vj * vj;
        for (int i = j + 1; i < m; ++i) vnorm2 += cj[i] * cj[i];
        if (vnorm2 == 0.0) {
            cj[j] = alpha;
            continue;
        }
        auto reflect = [&](double* x) {
            double s = vj * x[j];
            for (int i = j + 1; i < m; ++i) s += cj[i] * x[i];
            const double f = 2.0 * s / vnorm2;
            x[j] -= f * vj;
            for (int i = j + 1; i < m; ++i) x[i] -= f * cj[i];
        };
        for (int k = j + 1; k < n; ++k) reflect(col(k));
        reflect(qb.data());
        cj[j] = alpha;
    }

    // numerical rank relative to the largest pivot
    const double maxpivot = std::fabs(A[0]);
    int rank = 0;
    for (int j = 0; j < steps; ++j)
        if (std::fabs(col(j)[j]) > kRankTolerance * maxpivot) ++rank;

    auto Rij = [&](int i, int j) { return col(j)[i]; };
    std::vector<double> u(n, 0.0);
    if (rank > 0) {
        // h = R11^{-1} g
        std::vector<double> h(rank);
        for (int i = rank - 1; i >= 0; --i) {
            double s = qb[i];
            for (int k = i + 1; k < rank; ++k) s -= Rij(i, k) * h[k];
            h[i] = s / Rij(i, i);
        }
        if (rank == n) {
            u = h;
        } else {
            // minimum-norm branch: u1 = h - S u2, S = R11^{-1} R12,
            // (S^T S + I) u2 = S^T h
            const int q = n - rank;
            std::vector<double> S(static_cast<size_t>(rank) * q);
            for (int c2 = 0; c2 < q; ++c2)
                for (int i = rank - 1; i >= 0; --i) {
                    double s = Rij(i, rank + c2);
                    for (int k = i + 1; k < rank; ++k) s -= Rij(i, k) * S[static_cast<size_t>(k) * q + c2];
                    S[static_cast<size_t>(i) * q + c2] = s / Rij(i, i);
                }
            std::vector<double> M(static_cast<size_t>(q) * q, 0.0), rhs(q, 0.0);
            for (int a = 0; a < q; ++a) {
                for (int bq = 0; bq < q; ++bq) {
                    double s = a == bq ? 1.0 : 0.0;
                    for (int i = 0; i < rank; ++i)
                        s += S[static_cast<size_t>(i) * q + a] * S[static_cast<size_t>(i) * q + bq];
                    M[static_cast<size_t>(a) * q + bq] = s;
                }
                for (int i = 0; i < rank; ++i) rhs[a] += S[static_cast<size_t>(i) * q + a] * h[i];
            }
            // Cholesky solve (M is SPD)
            for (int a = 0; a < q; ++a) {
                for (int bq = 0; bq <= a; ++bq) {
                    double s = M[static_cast<size_t>(a) * q + bq];
                    for (int k = 0; k < bq; ++k)
                        s -= M[static_cast<size_t>(a) * q + k] * M[static_cast<size_t>(bq) * q + k];
                    M[static_cast<size_t>(a) * q + bq] =
                        a == bq ? std::sqrt(s) : s / M[static_cast<size_t>(bq) * q + bq];
                }
            }
            std::vector<double> z(q);
            for (int a = 0; a < q; ++a) {
                double s = rhs[a];
                for (int k = 0; k < a; ++k) s -= M[static_cast<size_t>(a) * q + k] * z[k];
                z[a] = s / M[static_cast<size_t>(a) * q + a];
            }
            for (int a = q - 1; a >= 0; --a) {
                double s = z[a];
                for (int k = a + 1; k < q; ++k) s -= M[static_cast<size_t>(k) * q + a] * z[k];
                z[a] = s / M[static_cast<size_t>(a) * q + a];
            }
            for (int i = 0; i < rank; ++i) {
                double s = h[i];
                for (int a = 0; a < q; ++a) s -= S[static_cast<size_t>(i) * q + a] * z[a];
                u[i] = s;
            }
            for (int a = 0; a < q; ++a) u[rank + a] = z[a];
        }
    }
    c.assign(n, 0.0);
    for (int j = 0; j < n; ++j) c[perm[j]] = u[j];

    // E = ||A c - b||^2 on the original matrix (approx.cpp:101)
    double e = 0.0;
    for (int i = 0; i < m; ++i) {
        double s = 0.0;
        for (int j = 0; j < n; ++j) s += A0[static_cast<size_t>(j) * m + i] * c[j];
        const double d = s - b0[i];
        e += d * d;
    }
    err = e;
    return true;
}

int fit_fixed(const double* samples, int R, int K, int T, std::vector<double>& c, double& err) {
    std::vector<double> A;
    if (!design_matrix(K, T, R, A))
        return fail(FBF_EINVAL, "design_matrix: invalid (K, T, R)");
    if (!fit_coefficients(A, 2 * R + 1, K, samples, c, err))
        return fail(FBF_EINVAL, "fit_coefficients: non-finite entries");
    return FBF_OK;
}

int scan(const double* samples, int R, int K, int t_max, int threads, std::vector<double>& errors) {
    if (t_max < 1) return fail(FBF_EINVAL, "period scan: t_max must be >= 1");
    if (K < 1 || K > 2 * R + 1) return fail(FBF_EINVAL, "period scan: invalid K");
    errors.assign(t_max, 0.0);
    std::vector<int> status(t_max, FBF_OK);
    parallel_for(1, t_max + 1, threads, [&](int T) {
        std::vector<double> A, c;
        double e = 0.0;
        design_matrix(K, T, R, A);
        if (!fit_coefficients(A, 2 * R + 1, K, samples, c, e)) status[T - 1] = FBF_EINVAL;
        errors[T - 1] = e;
    });
    for (int s : status)
        if (s != FBF_OK) return fail(s, "fit_coefficients: non-finite entries");
    return FBF_OK;
}

// approx.cpp:132-144 -- strict '<' keeps the smaller T on ties.
void argmin_period(const std::vector<double>& errors, int& T_best, double& e_best) {
    T_best = 1;
    e_best = errors[0];
    for (size_t T = 2; T <= errors.size(); ++T)
        if (errors[T - 1] < e_best) {
            T_best = static_cast<int>(T);
            e_best = errors[T - 1];
        }
}

// Where the period scans run: host threads (the reference's scan), or the GPU
// scan (fbf_scan.cu) followed by an exact host re-check of the near-minimal T.
struct ScanBackend {
    int threads = 1;
    int device = -1;  // < 0: host
    int cache_lo = 0, cache_n = 0, cache_tmax = 0;
    std::vector<double> cache;  // GPU errors of orders [cache_lo, cache_lo + cache_n)
};
// orders per GPU scan launch: the shared-memory footprint (and so the CTAs per
// SM) follows the largest order of a launch, so one order per launch
static const int kGpuOrderBatch = [] {
    const char* e = std::getenv("FBF_SCAN_BATCH");  // dev override
    return e ? std::max(1, std::atoi(e)) : 1;
}();
// relative window of the exact host re-check around the GPU minimum. GPU and host
// errors agree to ~1e-15 relative near the minimum and to ~1e-6 where the design
// matrix is ill-conditioned (large T, E far above the minimum); the runner-up T
// of the BASELINE configs is 0.09-1.6 % above the minimum
constexpr double kRecheckWindow = 1e-4;

// min_error_over_period (approx.cpp:132-144) through the backend. The GPU path
// re-evaluates every T whose GPU error is within kRecheckWindow of the GPU
// minimum with the host routine and takes the argmin of those exact values in
// ascending T, so (T_best, e_best) equal the host scan's.
int min_period(const double* samples, int R, int K, int t_max, ScanBackend& be, int& T_best, double& e_best) {
    if (be.device < 0 || K > gpu_scan_max_order(R)) {
        std::vector<double> errors;
        const int rc = scan(samples, R, K, t_max, be.threads, errors);
        if (rc != FBF_OK) return rc;
        argmin_period(errors, T_best, e_best);
        return FBF_OK;
    }
    if (t_max < 1) return fail(FBF_EINVAL, "period scan: t_max must be >= 1");
    if (K < 1 || K > 2 * R + 1) return fail(FBF_EINVAL, "period scan: invalid K");
    for (int i = 0; i < 2 * R + 1; ++i)
        if (!std::isfinite(samples[i])) return fail(FBF_EINVAL, "fit_coefficients: non-finite entries");
    if (!(K >= be.cache_lo && K < be.cache_lo + be.cache_n && be.cache_tmax == t_max)) {
        const int n = std::max(1, std::min(kGpuOrderBatch, gpu_scan_max_order(R) - K + 1));
        be.cache.assign(static_cast<size_t>(n) * t_max, 0.0);
        const int rc = gpu_scan_errors(samples, R, K, n, t_max, be.device, be.cache.data());
        if (rc != FBF_OK) {
            be.cache_n = 0;
            return rc;
        }
        be.cache_lo = K;
        be.cache_n = n;
        be.cache_tmax = t_max;
    }
    const double* eg = be.cache.data() + static_cast<size_t>(K - be.cache_lo) * t_max;
    double gmin = eg[0];
    for (int T = 2; T <= t_max; ++T) gmin = std::min(gmin, eg[T - 1]);
    const double limit = gmin + kRecheckWindow * std::fabs(gmin) + 1e-300;
    std::vector<int> cand;
    for (int T = 1; T <= t_max; ++T)
        if (eg[T - 1] <= limit) cand.push_back(T);
    if (cand.empty()) return fail(FBF_ECUDA, "gpu period scan: no finite error");
    // exact host errors of the candidates (many for flat scans, e.g. K = 1 where
    // E does not depend on T), on host threads; argmin in ascending T
    std::vector<double> ex(cand.size(), 0.0);
    std::vector<int> st(cand.size(), FBF_OK);
    parallel_for(0, static_cast<int>(cand.size()), cand.size() > 16 ? be.threads : 1, [&](int i) {
        std::vector<double> c;
        st[i] = fit_fixed(samples, R, K, cand[i], c, ex[i]);
    });
    for (size_t i = 0; i < cand.size(); ++i) {
        if (st[i] != FBF_OK) return fail(st[i], "fit_coefficients: non-finite entries");
        if (i == 0 || ex[i] < e_best) {
            T_best = cand[i];
            e_best = ex[i];
        }
    }
    return FBF_OK;
}

int copy_coeffs(const std::vector<double>& c, double* out, int cap) {
    if (static_cast<int>(c.size()) > cap)
        return fail(FBF_ECAPACITY, "coefficient buffer too small for K = " + std::to_string(c.size()));
    std::memcpy(out, c.data(), sizeof(double) * c.size());
    return FBF_OK;
}

int optimize_impl(const double* samples, int R, double tol, int t_max, int k_max, ScanBackend& be,
                  int* K_out, int* T_out, double* coeffs, int coeff_cap, double* err_out, double* per_order,
                  int* n_orders) {
    // approx.cpp:179-240
    if (!(tol > 0.0)) return fail(FBF_EINVAL, "optimize_parameters: tolerance must be positive");
    if (R < 1) return fail(FBF_EINVAL, "optimize_parameters: R must be >= 1");
    t_max = t_max > 0 ? t_max : 10 * R;
    k_max = k_max > 0 ? k_max : 2 * R + 1;
    if (k_max > 2 * R + 1) return fail(FBF_EINVAL, "optimize_parameters: k_max exceeds 2R+1");
    const int k_cap = std::min(k_max, t_max + 1);

    struct Order { int K, T; double e; };
    std::vector<Order> per;
    auto finish = [&](int K, int T, double e, int status, const std::string& msg) {
        std::vector<double> c;
        double e_fit = 0.0;
        const int rc = fit_fixed(samples, R, K, T, c, e_fit);
        if (rc != FBF_OK) return rc;
        const int rc2 = copy_coeffs(c, coeffs, coeff_cap);
        if (rc2 != FBF_OK) return rc2;
        if (K_out) *K_out = K;
        if (T_out) *T_out = T;
        if (err_out) *err_out = e;
        if (n_orders) *n_orders = static_cast<int>(per.size());
        if (per_order)
            for (size_t i = 0; i < per.size(); ++i) {
                per_order[3 * i] = per[i].K;
                per_order[3 * i + 1] = per[i].T;
                per_order[3 * i + 2] = per[i].e;
            }
        if (status != FBF_OK) return fail(status, msg);
        clear_error();
        return FBF_OK;
    };

    for (int K = 1; K <= k_cap; ++K) {
        int T = 1;
        double e = 0.0;
        const int rc = min_period(samples, R, K, t_max, be, T, e);
        if (rc != FBF_OK) return rc;
        per.push_back({K, T, e});
        if (e <= tol) return finish(K, T, e, FBF_OK, "");
    }
    // tolerance unreachable: best fit seen (min_element keeps the first minimum)
    size_t best = 0;
    for (size_t i = 1; i < per.size(); ++i)
        if (per[i].e < per[best].e) best = i;
    const std::string reason =
        k_cap < k_max
            ? "tolerance unreachable: the cosine span saturates at K = T_max + 1 = " +
                  std::to_string(k_cap)
            : "tolerance unreachable within K_max = " + std::to_string(k_max);
    return finish(per[best].K, per[best].T, per[best].e, FBF_EUNREACHABLE, reason);
}


int select_impl(int kind, double sigma, int R, double eps, int K, int T, int method_fbf, ScanBackend& be,
                int* K_out, int* T_out, double* coeffs, int coeff_cap, double* err_out) {
    // tools/fourierbf.cpp:185-234
    std::vector<double> b(static_cast<size_t>(2 * R + 1));
    if (R < 1) return fail(FBF_EINVAL, "range kernel: dynamic range must be >= 1");
    int rc = fbf_sample_range_kernel(kind, sigma, R, b.data());
    if (rc != FBF_OK) return rc;
    const bool has_eps = eps > 0.0, has_K = K > 0, has_T = T > 0;
    if (has_eps && (has_K || has_T))
        return fail(FBF_EINVAL, "--eps and --K/--T are mutually exclusive");

    auto fixed = [&](int k, int t) {
        std::vector<double> c;
        double e = 0.0;
        int r2 = fit_fixed(b.data(), R, k, t, c, e);
        if (r2 != FBF_OK) return r2;
        r2 = copy_coeffs(c, coeffs, coeff_cap);
        if (r2 != FBF_OK) return r2;
        if (K_out) *K_out = k;
        if (T_out) *T_out = t;
        if (err_out) *err_out = e;
        clear_error();
        return FBF_OK;
    };

    if (method_fbf) {
        // fixed-period baseline: T = R, K given directly or matched via eps
        int k = K;
        if (!has_K) {
            if (!has_eps) return fail(FBF_EINVAL, "fbf needs --K or --eps");
            std::vector<double> tmp(static_cast<size_t>(2 * R + 1));
            int k_star = 0, t_star = 0;
            double e = 0.0;
            rc = optimize_impl(b.data(), R, eps, 0, 0, be, &k_star, &t_star, tmp.data(),
                               static_cast<int>(tmp.size()), &e, nullptr, nullptr);
            if (rc != FBF_OK) return rc;
            k = k_star;
        }
        return fixed(k, R);
    }
    if (has_K) {
        int t = T;
        if (!has_T) {
            double eb = 0.0;
            rc = min_period(b.data(), R, K, 10 * R, be, t, eb);
            if (rc != FBF_OK) return rc;
        }
        return fixed(K, t);
    }
    if (has_T) return fail(FBF_EINVAL, "--T needs --K");
    if (!has_eps) return fail(FBF_EINVAL, "need --eps or --K");
    return optimize_impl(b.data(), R, eps, 0, 0, be, K_out, T_out, coeffs, coeff_cap, err_out, nullptr,
                         nullptr);
}

}  // namespace

void set_error(const std::string& msg) { g_last_error = msg; }
void clear_error() { g_last_error.clear(); }
int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}
const char* last_error_cstr() { return g_last_error.c_str(); }

}  // namespace fbf_b200

using namespace fbf_b200;

extern "C" {

const char* fbf_last_error(void) { return fbf_b200::last_error_cstr(); }

int fbf_build_spatial_kernel(double theta, double* taps, int cap) {
    // kernels.cpp:105-118
    if (!(theta > 0.0) || !std::isfinite(theta))
        return -fail(FBF_EINVAL, "spatial kernel: theta must be positive");
    const int r = static_cast<int>(std::ceil(3.0 * theta));
    if (2 * r + 1 > cap) return -fail(FBF_ECAPACITY, "spatial kernel: tap buffer too small");
    for (int j = 0; j <= r; ++j) {
        const double v = std::exp(-(static_cast<double>(j) * j) / (2.0 * theta * theta));
        taps[r + j] = v;
        taps[r - j] = v;
    }
    return r;
}

int fbf_sample_range_kernel(int kind, double sigma, int R, double* values) {
    // kernels.cpp:11-32 (validate_parametric, evaluate_kind) and :78-103
    if (!(sigma > 0.0) || !std::isfinite(sigma))
        return fail(FBF_EINVAL, "range kernel: sigma must be positive");
    if (R < 1) return fail(FBF_EINVAL, "range kernel: dynamic range must be >= 1");
    for (int t = 0; t <= R; ++t) {
        const double x = static_cast<double>(t);
        double v;
        switch (kind) {
        case FBF_KERNEL_GAUSSIAN: v = std::exp(-(x * x) / (2.0 * sigma * sigma)); break;
        case FBF_KERNEL_EXPONENTIAL: v = std::exp(-std::abs(x) / sigma); break;
        case FBF_KERNEL_CAUCHY: v = 1.0 / (1.0 + (x * x) / (sigma * sigma)); break;
        default: return fail(FBF_EINVAL, "range kernel: unknown kind");
        }
        values[R + t] = v;
        values[R - t] = v;
    }
    return FBF_OK;
}

double fbf_frequency_of(int half_period) {
    return 2.0 * std::numbers::pi / (2.0 * half_period + 1.0);  // approx.cpp:17-19
}

int fbf_fit_fixed_period(const double* samples, int R, int K, int T, double* coeffs,
                         double* err_out) {
    std::vector<double> c;
    double e = 0.0;
    const int rc = fit_fixed(samples, R, K, T, c, e);
    if (rc != FBF_OK) return rc;
    std::memcpy(coeffs, c.data(), sizeof(double) * K);
    if (err_out) *err_out = e;
    return FBF_OK;
}

int fbf_scan_period_errors(const double* samples, int R, int K, int t_max, int threads,
                           double* errors) {
    std::vector<double> e;
    const int rc = scan(samples, R, K, t_max, threads, e);
    if (rc != FBF_OK) return rc;
    std::memcpy(errors, e.data(), sizeof(double) * e.size());
    return FBF_OK;
}

int fbf_min_error_over_period(const double* samples, int R, int K, int t_max, int threads,
                              int* T_best, double* err_out) {
    std::vector<double> e;
    const int rc = scan(samples, R, K, t_max, threads, e);
    if (rc != FBF_OK) return rc;
    int T = 1;
    double eb = 0.0;
    argmin_period(e, T, eb);
    if (T_best) *T_best = T;
    if (err_out) *err_out = eb;
    return FBF_OK;
}

int fbf_optimize_parameters(const double* samples, int R, double tol, int t_max, int k_max,
                            int threads, int* K_out, int* T_out, double* coeffs, int coeff_cap,
                            double* err_out, double* per_order, int* n_orders) {
    ScanBackend be;
    be.threads = threads;
    return optimize_impl(samples, R, tol, t_max, k_max, be, K_out, T_out, coeffs, coeff_cap, err_out, per_order,
                         n_orders);
}

int fbf_optimize_parameters_gpu(const double* samples, int R, double tol, int t_max, int k_max, int device,
                                int* K_out, int* T_out, double* coeffs, int coeff_cap, double* err_out,
                                double* per_order, int* n_orders) {
    ScanBackend be;
    be.device = device;
    be.threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    return optimize_impl(samples, R, tol, t_max, k_max, be, K_out, T_out, coeffs, coeff_cap, err_out, per_order,
                         n_orders);
}

int fbf_select_params(int kind, double sigma, int R, double eps, int K, int T, int method_fbf,
                      int threads, int* K_out, int* T_out, double* coeffs, int coeff_cap,
                      double* err_out) {
    ScanBackend be;
    be.threads = threads;
    return select_impl(kind, sigma, R, eps, K, T, method_fbf, be, K_out, T_out, coeffs, coeff_cap, err_out);
}

int fbf_select_params_gpu(int kind, double sigma, int R, double eps, int K, int T, int method_fbf, int device,
                          int* K_out, int* T_out, double* coeffs, int coeff_cap, double* err_out) {
    ScanBackend be;
    be.device = device;
    be.threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    return select_impl(kind, sigma, R, eps, K, T, method_fbf, be, K_out, T_out, coeffs, coeff_cap, err_out);
}

int fbf_scan_period_errors_gpu(const double* samples, int R, int K_lo, int nK, int t_max, int device,
                               double* errors) {
    const int rc = gpu_scan_errors(samples, R, K_lo, nK, t_max, device, errors);
    if (rc == FBF_OK) clear_error();
    return rc;
}

int fbf_min_error_over_period_gpu(const double* samples, int R, int K, int t_max, int device, int* T_best,
                                  double* err_out) {
    ScanBackend be;
    be.device = device;
    be.threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    int T = 1;
    double e = 0.0;
    const int rc = min_period(samples, R, K, t_max, be, T, e);
    if (rc != FBF_OK) return rc;
    if (T_best) *T_best = T;
    if (err_out) *err_out = e;
    clear_error();
    return FBF_OK;
}

// lut.cpp:61-113 -- K*, T* per (sigma, eps) cell (Gaussian kernel), row-major
// [n_sigma][n_eps]; device >= 0 runs the period scans on the GPU (same cells).
int fbf_build_lut(const double* sigmas, int n_sigma, const double* epsilons, int n_eps, int R, int t_max,
                  int device, int threads, int* K_out, int* T_out) {
    if (n_sigma < 2) return fail(FBF_EINVAL, "LUT: sigma grid needs at least two points");
    for (int i = 1; i < n_sigma; ++i)
        if (!(sigmas[i] > sigmas[i - 1])) return fail(FBF_EINVAL, "LUT: sigma grid must be strictly ascending");
    for (int i = 0; i < n_sigma; ++i)
        if (!(sigmas[i] > 0.0)) return fail(FBF_EINVAL, "LUT: sigma values must be positive");
    if (n_eps < 2) return fail(FBF_EINVAL, "LUT: eps grid needs at least two points");
    std::vector<double> logeps(n_eps);
    for (int j = 0; j < n_eps; ++j) {
        if (!(epsilons[j] > 0.0) || !(epsilons[j] < 1.0)) return fail(FBF_EINVAL, "LUT: eps values must be in (0, 1)");
        logeps[j] = std::log10(1.0 / epsilons[j]);
    }
    for (int j = 1; j < n_eps; ++j)
        if (!(logeps[j] > logeps[j - 1]))
            return fail(FBF_EINVAL, "LUT: log10(1/eps) grid must be strictly ascending");
    if (R < 1) return fail(FBF_EINVAL, "range kernel: dynamic range must be >= 1");
    const int cells = n_sigma * n_eps;
    std::vector<int> status(cells, FBF_OK);
    std::vector<std::string> msg(cells);
    auto cell = [&](int c) {
        const int i = c / n_eps, j = c % n_eps;
        std::vector<double> b(2 * R + 1), coeffs(2 * R + 1);
        int rc = fbf_sample_range_kernel(FBF_KERNEL_GAUSSIAN, sigmas[i], R, b.data());
        ScanBackend be;
        be.threads = device >= 0 ? std::max(1, threads) : 1;
        be.device = device;
        double e = 0.0;
        if (rc == FBF_OK)
            rc = optimize_impl(b.data(), R, epsilons[j], t_max, 0, be, &K_out[c], &T_out[c], coeffs.data(),
                               static_cast<int>(coeffs.size()), &e, nullptr, nullptr);
        status[c] = rc;
        if (rc != FBF_OK) msg[c] = last_error_cstr();
    };
    if (device >= 0) {
        for (int c = 0; c < cells; ++c) cell(c);  // one GPU: cells in order, each scan on the device
    } else {
        parallel_for(0, cells, threads, cell);   // lut.cpp:87-105
    }
    for (int c = 0; c < cells; ++c)
        if (status[c] != FBF_OK) {
            char buf[128];
            std::snprintf(buf, sizeof buf, "LUT build failed at cell sigma=%.17g eps=%.17g: ", sigmas[c / n_eps],
                          epsilons[c % n_eps]);
            return fail(status[c] == FBF_EUNREACHABLE ? FBF_EUNREACHABLE : status[c], buf + msg[c]);
        }
    clear_error();
    return FBF_OK;
}

// lut.cpp:116-143 -- bilinear in (sigma, log10(1/eps)); K rounds up, T to nearest.
int fbf_query_lut(const double* sigma_grid, int n_sigma, const double* logeps_grid, int n_eps, const int* K,
                  const int* T, double sigma, double eps, int* K_out, int* T_out) {
    if (n_sigma < 2 || n_eps < 2) return fail(FBF_EINVAL, "LUT: malformed table");
    if (!(eps > 0.0) || !(eps < 1.0)) return fail(FBF_ERANGE, "LUT query: eps must be in (0, 1)");
    const double le = std::log10(1.0 / eps);
    if (sigma < sigma_grid[0] || sigma > sigma_grid[n_sigma - 1] || le < logeps_grid[0] ||
        le > logeps_grid[n_eps - 1])
        return fail(FBF_ERANGE, "LUT query: (sigma, eps) outside the table grid");
    auto locate = [](const double* g, int n, double x) {
        const int i = static_cast<int>(std::upper_bound(g, g + n, x) - g);
        return std::min(i > 0 ? i - 1 : 0, n - 2);
    };
    const int i = locate(sigma_grid, n_sigma, sigma), j = locate(logeps_grid, n_eps, le);
    const double tx = (sigma - sigma_grid[i]) / (sigma_grid[i + 1] - sigma_grid[i]);
    const double ty = (le - logeps_grid[j]) / (logeps_grid[j + 1] - logeps_grid[j]);
    auto lerp = [](double a, double b, double t) { return a + t * (b - a); };
    auto bilinear = [&](const int* g) {
        const double lo = lerp(g[i * n_eps + j], g[i * n_eps + j + 1], ty);
        const double hi = lerp(g[(i + 1) * n_eps + j], g[(i + 1) * n_eps + j + 1], ty);
        return lerp(lo, hi, tx);
    };
    *K_out = static_cast<int>(std::ceil(bilinear(K)));
    *T_out = static_cast<int>(std::lround(bilinear(T)));
    clear_error();
    return FBF_OK;
}

int fbf_scan_gpu_max_order(int R) { return R >= 1 ? gpu_scan_max_order(R) : 0; }

}  // extern "C"
