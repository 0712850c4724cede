// fbf_internal.h -- shared declarations of the fbf host library (not part of the ABI).
#pragma once

#include <mutex>
#include <string>

namespace fbf_b200 {

// Thread-local last-error message behind fbf_last_error().
void set_error(const std::string& msg);
void clear_error();
int fail(int code, const std::string& msg);

// Per-device context of the filter library (fbf_api.cu): its compute stream
// (a cudaStream_t) and the mutex that serialises work on it.
int device_context(int device, void** stream, std::mutex** mtx);
// Counts one launch of an fbf kernel (fbf_kernel_launches()).
void count_launch(unsigned long long n = 1);

// GPU period scan (fbf_scan.cu): errors[(K - K_lo) * t_max + T - 1] = E(K, T)
// for K in [K_lo, K_lo + nK), T in [1, t_max]; FP64, ~1e-12 relative to the
// host scan. gpu_scan_max_order(R): largest K the kernel takes.
int gpu_scan_errors(const double* samples, int R, int K_lo, int nK, int t_max, int device, double* errors);
int gpu_scan_max_order(int R);

// Runs fn(i) for i in [begin, end) over at most `threads` std::threads, each
// owning a contiguous chunk (the reference's parallel_for,
// include/fourierbf/parallel.hpp:16-52): outputs are disjoint, so results do
// not depend on the thread count.
template <typename Fn>
void parallel_for(int begin, int end, int threads, Fn&& fn);

}  // namespace fbf_b200

#include <algorithm>
#include <thread>
#include <vector>

namespace fbf_b200 {
template <typename Fn>
void parallel_for(int begin, int end, int threads, Fn&& fn) {
    const int n = end - begin;
    if (n <= 0) return;
    threads = std::clamp(threads, 1, n);
    if (threads == 1) {
        for (int i = begin; i < end; ++i) fn(i);
        return;
    }
    std::vector<std::thread> workers;
    const int chunk = (n + threads - 1) / threads;
    for (int w = 0; w < threads; ++w) {
        const int lo = begin + w * chunk, hi = std::min(lo + chunk, end);
        if (lo >= hi) break;
        workers.emplace_back([lo, hi, &fn] {
            for (int i = lo; i < hi; ++i) fn(i);
        });
    }
    for (auto& t : workers) t.join();
}
}  // namespace fbf_b200
