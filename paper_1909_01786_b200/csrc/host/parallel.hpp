// Host parallelism for the load path (parse -> completion -> store build):
// plain std::thread fork-join over index ranges. Small inputs stay on the
// calling thread (a thread start costs tens of microseconds).
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <exception>
#include <thread>
#include <vector>

namespace yas {

inline unsigned host_threads() {
    static const unsigned n = [] {
        const unsigned hw = std::thread::hardware_concurrency();
        return std::max(1u, std::min(hw ? hw : 1u, 32u));
    }();
    return n;
}

/// fn(chunk, begin, end) over `parts` contiguous chunks of [0, n), one thread each
/// (parts = 1 below `grain` items). Exceptions are rethrown on the caller.
template <class F>
void parallel_chunks(std::size_t n, std::size_t grain, F&& fn, unsigned parts = 0) {
    if (parts == 0) parts = host_threads();
    if (n < grain || parts <= 1) parts = 1;
    parts = static_cast<unsigned>(std::min<std::size_t>(parts, std::max<std::size_t>(1, n)));
    if (parts == 1) {
        fn(0u, std::size_t{0}, n);
        return;
    }
    std::vector<std::thread> th;
    std::vector<std::exception_ptr> err(parts);
    const std::size_t step = (n + parts - 1) / parts;
    for (unsigned c = 1; c < parts; ++c)
        th.emplace_back([&, c] {
            try {
                fn(c, std::min(n, c * step), std::min(n, (c + 1) * step));
            } catch (...) {
                err[c] = std::current_exception();
            }
        });
    try {
        fn(0u, std::size_t{0}, std::min(n, step));
    } catch (...) {
        err[0] = std::current_exception();
    }
    for (std::thread& t : th) t.join();
    for (auto& e : err)
        if (e) std::rethrow_exception(e);
}

/// Number of chunks parallel_chunks will use for (n, grain).
inline unsigned chunk_count(std::size_t n, std::size_t grain) {
    const unsigned parts = host_threads();
    if (n < grain || parts <= 1) return 1;
    return static_cast<unsigned>(std::min<std::size_t>(parts, std::max<std::size_t>(1, n)));
}

/// In place exclusive prefix sum; returns the total.
template <class T>
T exclusive_scan_inplace(std::vector<T>& v) {
    T run = 0;
    for (T& x : v) {
        const T y = x;
        x = run;
        run += y;
    }
    return run;
}

}  // namespace yas
