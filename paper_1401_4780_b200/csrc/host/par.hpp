// Host-side data parallelism for the drop-in path's O(nnz) passes (CSR
// assembly from coordinate arrays, row norms, normalization): f(t, lo, hi)
// over contiguous chunks of [0, n) on up to 16 threads. Small inputs run on
// the caller.
#pragma once
#include <algorithm>
#include <cstddef>
#include <thread>
#include <vector>

namespace asyrk::par {

inline int threads_for(std::size_t n) {
    constexpr std::size_t kMinChunk = 1u << 16;
    const unsigned hc = std::max(1u, std::thread::hardware_concurrency());
    return (int)std::max<std::size_t>(1, std::min<std::size_t>({(std::size_t)std::min(hc, 16u), n / kMinChunk + 1}));
}

template <class F>
void chunks(std::size_t n, int T, F&& f) {
    if (T <= 1) {
        f(0, std::size_t{0}, n);
        return;
    }
    std::vector<std::thread> ts;
    ts.reserve((std::size_t)T - 1);
    for (int t = 1; t < T; ++t) ts.emplace_back([&, t] { f(t, n * (std::size_t)t / (std::size_t)T, n * ((std::size_t)t + 1) / (std::size_t)T); });
    f(0, std::size_t{0}, n / (std::size_t)T);
    for (auto& th : ts) th.join();
}

}  // namespace asyrk::par
