// Fixed-theta synthetic systems for the BASELINE configs (include/asyrk_datagen.h).
#include "asyrk_datagen.h"

#include <algorithm>
#include <cmath>
#include <thread>
#include <vector>

#include "asyrk_cuda.h"

namespace {

inline uint64_t mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// xoshiro256** (Blackman & Vigna)
struct Xoshiro {
    uint64_t s[4];
    Xoshiro(uint64_t seed, uint64_t stream) {
        uint64_t z = mix64(seed) ^ mix64(stream + 0x632BE59BD9B4E019ULL);
        for (auto& w : s) w = z = mix64(z);
    }
    static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
    uint64_t next() {
        const uint64_t r = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
        s[2] ^= s[0];
        s[3] ^= s[1];
        s[1] ^= s[2];
        s[0] ^= s[3];
        s[2] ^= t;
        s[3] = rotl(s[3], 45);
        return r;
    }
    uint64_t below(uint64_t n) {  // unbiased (rejection)
        const uint64_t lim = UINT64_MAX - UINT64_MAX % n;
        for (;;) {
            const uint64_t v = next();
            if (v < lim) return v % n;
        }
    }
    double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    double normal() {
        for (;;) {
            const double u = 2.0 * unit() - 1.0, v = 2.0 * unit() - 1.0, q = u * u + v * v;
            if (q < 1.0 && q != 0.0) return u * std::sqrt(-2.0 * std::log(q) / q);
        }
    }
};

template <class F>
void parallel_rows(int64_t rows, int threads, F&& f) {
    if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
    threads = (int)std::min<int64_t>(threads, std::max<int64_t>(1, rows / 1024));
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
        const int64_t lo = rows * t / threads, hi = rows * (t + 1) / threads;
        pool.emplace_back([&f, lo, hi] { f(lo, hi); });
    }
    for (auto& th : pool) th.join();
}

}  // namespace

extern "C" int asyrk_generate_fixed_theta(int64_t m, int64_t n, int64_t theta, uint64_t seed, int32_t value_dist,
                                          double scale_decades, int64_t k, int32_t threads, int64_t* row_ptr,
                                          int64_t* col_idx, double* values, double* row_norm, double* b,
                                          double* x_star, int32_t* normalized) {
    if (m < 1 || n < 1 || theta < 1 || theta > n || k < 1) return ASYRK_E_InvalidArgument;
    // X* first: its own streams, one per row of X*
    parallel_rows(n, threads, [&](int64_t lo, int64_t hi) {
        for (int64_t j = lo; j < hi; ++j) {
            Xoshiro g(seed ^ 0x5EEDF00DULL, 0x8000000000000000ULL | (uint64_t)j);
            for (int64_t c = 0; c < k; ++c) x_star[j * k + c] = g.normal();
        }
    });
    std::vector<char> row_unit((size_t)m, 1);
    parallel_rows(m, threads, [&](int64_t lo, int64_t hi) {
        std::vector<int64_t> cols((size_t)theta);
        for (int64_t i = lo; i < hi; ++i) {
            Xoshiro g(seed, (uint64_t)i);
            // theta distinct columns (rejection against the row so far), sorted
            for (int64_t t = 0; t < theta;) {
                const int64_t c = (int64_t)g.below((uint64_t)n);
                if (std::find(cols.begin(), cols.begin() + t, c) == cols.begin() + t) cols[(size_t)t++] = c;
            }
            std::sort(cols.begin(), cols.end());
            const int64_t base = i * theta;
            row_ptr[i + 1] = base + theta;
            double ss = 0.0;
            for (int64_t t = 0; t < theta; ++t) {
                double v;
                do {
                    v = value_dist == ASYRK_GEN_UNIFORM ? 2.0 * g.unit() - 1.0 : g.normal();
                } while (v == 0.0);
                col_idx[base + t] = cols[(size_t)t];
                values[base + t] = v;
                ss += v * v;
            }
            // normalize_rows semantics (ref csr.cpp:113-138)
            double nrm = std::sqrt(ss);
            if (std::abs(nrm - 1.0) > 1e-12) {
                for (int64_t t = 0; t < theta; ++t) values[base + t] /= nrm;
                ss = 0.0;
                for (int64_t t = 0; t < theta; ++t) ss += values[base + t] * values[base + t];
                nrm = std::sqrt(ss);
            }
            if (scale_decades > 0.0) {
                const double s = std::pow(10.0, scale_decades * (2.0 * g.unit() - 1.0));
                ss = 0.0;
                for (int64_t t = 0; t < theta; ++t) {
                    values[base + t] *= s;
                    ss += values[base + t] * values[base + t];
                }
                nrm = std::sqrt(ss);
            }
            row_norm[i] = nrm;
            row_unit[(size_t)i] = std::abs(nrm - 1.0) <= 1e-12;
            // B = A X* in storage order (row_dot, ref csr.cpp:65-70)
            for (int64_t c = 0; c < k; ++c) {
                double s = 0.0;
                for (int64_t t = 0; t < theta; ++t) s += values[base + t] * x_star[col_idx[base + t] * k + c];
                b[i * k + c] = s;
            }
        }
    });
    row_ptr[0] = 0;
    int32_t all = 1;
    for (int64_t i = 0; i < m; ++i)
        if (!row_unit[(size_t)i]) {
            all = 0;
            break;
        }
    if (normalized) *normalized = all;
    return 0;
}
