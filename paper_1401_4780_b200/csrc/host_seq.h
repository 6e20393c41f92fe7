// Host side of the deterministic mode: the reference's seeded row sequence.
//
// The reference defines its randomness completely (ref/include/asyrk/rng.hpp):
// stream s of seed b is std::mt19937_64 seeded with splitmix64(b ^ s)
// (rng.hpp:14-22), integers come from rejection sampling (rng.hpp:26-33),
// permutations from Fisher-Yates run from the top (rng.hpp:51-57) applied
// cumulatively per epoch (parallel.cpp:119-123,160-162; kaczmarz.cpp:157-160,
// 203), norm-proportional rows from a Walker alias table built with
// small/large stacks popped from the back (kaczmarz.cpp:14-61). The
// deterministic GPU worker (det.cu) consumes exactly this sequence, so it is
// produced here, chunk by chunk, overlapped with the GPU's work on the
// previous chunk. std::mt19937_64 is fully specified by the C++ standard.
#pragma once
#include <cmath>
#include <cstdint>
#include <random>
#include <stdexcept>
#include <vector>

namespace ak {

inline uint64_t splitmix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

class RefStream {
  public:
    RefStream(uint64_t seed, uint64_t stream) : g_(splitmix64(seed ^ stream)) {}
    uint64_t raw() { return g_(); }
    // rejection then modulo, rng.hpp:26-33
    uint64_t below(uint64_t n) {
        const uint64_t lim = UINT64_MAX - UINT64_MAX % n;
        for (;;) {
            const uint64_t v = g_();
            if (v < lim) return v % n;
        }
    }
    // top 53 bits, rng.hpp:36-38
    double unit() { return static_cast<double>(g_() >> 11) * 0x1.0p-53; }
    // polar Box-Muller, rng.hpp:41-48
    double normal() {
        for (;;) {
            const double u = 2.0 * unit() - 1.0, v = 2.0 * unit() - 1.0;
            const double s = u * u + v * v;
            if (s < 1.0 && s != 0.0) return u * std::sqrt(-2.0 * std::log(s) / s);
        }
    }
    template <class I>
    void shuffle(std::vector<I>& p) {
        for (std::size_t i = p.size(); i > 1; --i) {
            const std::size_t j = static_cast<std::size_t>(below(i));
            std::swap(p[i - 1], p[j]);
        }
    }

  private:
    std::mt19937_64 g_;
};

// Walker alias table with the reference's construction order.
struct HostAlias {
    std::vector<double> prob;
    std::vector<int32_t> alias;

    // returns false on an invalid weight vector (InvalidArgument upstream)
    bool build(const std::vector<double>& w) {
        const std::size_t n = w.size();
        if (n == 0) return false;
        double sum = 0.0;
        for (double v : w) {
            if (!(v >= 0.0)) return false;
            sum += v;
        }
        if (sum <= 0.0) return false;
        prob.assign(n, 0.0);
        alias.assign(n, 0);
        std::vector<double> sc(n);
        for (std::size_t k = 0; k < n; ++k) sc[k] = w[k] * static_cast<double>(n) / sum;
        std::vector<int32_t> small, large;
        small.reserve(n);
        large.reserve(n);
        for (std::size_t k = 0; k < n; ++k) (sc[k] < 1.0 ? small : large).push_back(static_cast<int32_t>(k));
        while (!small.empty() && !large.empty()) {
            const int32_t s = small.back();
            small.pop_back();
            const int32_t l = large.back();
            prob[s] = sc[s];
            alias[s] = l;
            sc[l] -= 1.0 - sc[s];
            if (sc[l] < 1.0) {
                large.pop_back();
                small.push_back(l);
            }
        }
        for (int32_t k : large) prob[k] = 1.0;
        for (int32_t k : small) prob[k] = 1.0;
        return true;
    }
    int32_t sample(RefStream& g) const {
        const int32_t k = static_cast<int32_t>(g.below(prob.size()));
        const double u = g.unit();
        return u < prob[k] ? k : alias[k];
    }
};

// Row-sequence generator for one deterministic solve.
//   mode 0: uniform (with replacement)   kaczmarz.cpp:205-208 / parallel.cpp:165-166
//   mode 1: norm_proportional (alias)    kaczmarz.cpp:209-213
//   mode 2: cumulative shuffle           kaczmarz.cpp:203,214-217 / parallel.cpp:160-164
// with_picks: single_component draws its component right after each row
// (parallel.cpp:183-185), from the same stream.
class SeqGen {
  public:
    SeqGen(uint64_t seed, int mode, int64_t m, const std::vector<int32_t>* row_len, const HostAlias* alias,
           bool with_picks)
        : g_(seed, 0), mode_(mode), m_(m), row_len_(row_len), alias_(alias), picks_(with_picks) {
        if (mode_ == 2) {
            perm_.resize(static_cast<std::size_t>(m));
            for (int64_t i = 0; i < m; ++i) perm_[static_cast<std::size_t>(i)] = static_cast<int32_t>(i);
        }
    }
    // One epoch (m row events) appended at seq/picks.
    void epoch(int32_t* seq, int32_t* picks) {
        if (mode_ == 2) g_.shuffle(perm_);
        for (int64_t q = 0; q < m_; ++q) {
            int32_t i;
            if (mode_ == 0)
                i = static_cast<int32_t>(g_.below(static_cast<uint64_t>(m_)));
            else if (mode_ == 1)
                i = alias_->sample(g_);
            else
                i = perm_[static_cast<std::size_t>(q)];
            seq[q] = i;
            if (picks_) picks[q] = static_cast<int32_t>(g_.below(static_cast<uint64_t>((*row_len_)[i])));
        }
    }

  private:
    RefStream g_;
    int mode_;
    int64_t m_;
    const std::vector<int32_t>* row_len_;
    const HostAlias* alias_;
    bool picks_;
    std::vector<int32_t> perm_;
};

}  // namespace ak
