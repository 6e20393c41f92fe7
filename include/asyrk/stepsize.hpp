// Drop-in step-size corollary (ref/include/asyrk/stepsize.hpp:10-45, scalar
// host math): the tau-feasibility 2e*lambda_max*(tau+1)/m <= 1 that the
// active-warp sweep reports beside each warp count.
#pragma once

#include <optional>

#include "asyrk/stats.hpp"

namespace asyrk {

struct GammaBounds {
    double b1 = 0.0;
    double b2 = 0.0;
    double b3 = 0.0;
    double gamma = 0.0;
};

struct StepParams {
    index_t tau = 0;
    double rho = 0.0;
    double psi = 0.0;
    double gamma = 0.0;
    GammaBounds gamma_bounds;
    bool feasible = false;
    std::optional<double> rate_iter;
    std::optional<double> rate_simplified;
};

struct ProbBound {
    double epsilon = 0.0;
    double eta = 0.0;
    index_t j_min = 0;
};

struct RateIteration {
    double per_iteration = 0.0;  // 1 - lambda_min*gamma*(2-gamma*psi)/m
    double per_epoch = 0.0;      // per_iteration^m
};

double psi(double mu, double lambda_max, index_t tau, double rho, index_t m);
GammaBounds gamma_bounds(const SystemStats& stats, index_t tau, double rho);
StepParams corollary_params(const SystemStats& stats, index_t tau);

/// ref stepsize.hpp:49-58 / stepsize.cpp:84-125 (needs lambda_min: the
/// dense spectrum of compute_stats' exact_spectral)
RateIteration rate_iteration(const SystemStats& stats, double gamma, double psi_value);
ProbBound iteration_bound(const SystemStats& stats, double x0_dist_sq, double epsilon, double eta);

/// Largest tau with 2e*lambda_max*(tau+1)/m <= 1 (PAPER §4 Corollary), i.e.
/// floor(m / (2e*lambda_max)) - 1; negative when even tau = 0 is infeasible.
index_t max_feasible_tau(index_t m, double lambda_max);

}  // namespace asyrk
