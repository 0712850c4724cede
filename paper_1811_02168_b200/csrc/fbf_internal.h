// fbf_internal.h -- shared declarations of the fbf host library (not part of the ABI).
#pragma once

#include <string>

namespace fbf_b200 {

// Thread-local last-error message behind fbf_last_error().
void set_error(const std::string& msg);
void clear_error();
int fail(int code, const std::string& msg);

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
