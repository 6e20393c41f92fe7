// Drop-in serial RK entry point (ref/include/asyrk/kaczmarz.hpp:20-115, hot-path
// subset). rk_solve runs on the GPU's deterministic worker and reproduces the
// reference's iterates bit for bit.
#pragma once

#include <cstdint>
#include <random>
#include <span>
#include <vector>

#include "asyrk/csr.hpp"
#include "asyrk/rng.hpp"
#include "asyrk/trace.hpp"

namespace asyrk {

class SolutionProjector;  // dense oracle (asyrk/dense.hpp); its distance runs on the device as x_star = A^+ b

inline constexpr index_t kAllComponents = -1;

enum class UpdateVariant { single_component, full_row };

/// What one update event touches (ref kaczmarz.hpp:22-29).
struct UpdateEvent {
    index_t j = 0;                // iteration index
    index_t i = 0;                // selected row
    index_t t = kAllComponents;   // selected component, kAllComponents for the row
    index_t k = 0;                // iterate index the residual was read from
    double step = 0.0;            // single component: the increment; row: the multiplier c
};

/// Walker alias sampler over a fixed nonnegative weight vector
/// (ref kaczmarz.hpp:32-41); the construction order matches the reference so
/// seeded draws are identical.
class AliasTable {
  public:
    explicit AliasTable(std::span<const double> weights);
    index_t sample(std::mt19937_64& gen) const;
    index_t size() const { return static_cast<index_t>(prob_.size()); }

  private:
    std::vector<double> prob_;
    std::vector<index_t> alias_;
};

enum class Sampling {
    uniform,            // rows equiprobable; requires normalized A
    norm_proportional,  // P(i) proportional to ||a_i||^2, alias table
    shuffle,            // per-epoch random permutation, each row once
};

struct RkConfig {
    index_t max_epochs = 100;
    double target_r_sq = 0.0;
    std::uint64_t seed = 0;
    Sampling sampling = Sampling::uniform;
    const std::vector<double>* x_star = nullptr;
    const SolutionProjector* projector = nullptr;
};

Trace rk_solve(const CsrMatrix& A, std::span<const double> b, std::span<const double> x0, const RkConfig& cfg);

}  // namespace asyrk
