// power_iteration_lambda_max on the device (ref/src/stats.cpp:15-50) and the
// step-size corollary (ref/src/stepsize.cpp:26-82), scalar host math.
#include <algorithm>
#include <cmath>
#include <numbers>

#include "asyrk/error.hpp"
#include "asyrk/stepsize.hpp"
#include "asyrk_cuda.h"

namespace asyrk {

double power_iteration_lambda_max(const CsrMatrix& A, double tol, index_t max_iters) {
    double lam = 0.0;
    int64_t iters = 0;
    throw_status(asyrk_system_power_iteration(A.device(0), tol, max_iters, &lam, &iters));
    return lam;
}

double psi(double mu, double lambda_max, index_t tau, double rho, index_t m) {
    if (m < 1) fail(ErrorCode::InvalidArgument, "m must be >= 1");
    if (tau < 0) fail(ErrorCode::InvalidArgument, "tau must be >= 0");
    if (tau == 0) return mu;
    if (!(rho > 1.0)) fail(ErrorCode::InvalidRho, "rho must exceed 1 when tau > 0");
    const double t = static_cast<double>(tau);
    return mu + 2.0 * lambda_max * t * std::pow(rho, t) / static_cast<double>(m);
}

static void need_core(const SystemStats& s) {
    if (s.m <= 0 || s.mu <= 0 || s.alpha <= 0.0 || s.lambda_max <= 0.0)
        fail(ErrorCode::MissingStats, "need m, mu, alpha and lambda_max to evaluate step bounds");
}

GammaBounds gamma_bounds(const SystemStats& s, index_t tau, double rho) {
    need_core(s);
    if (!(rho > 1.0)) fail(ErrorCode::InvalidRho, "rho must exceed 1");
    const double m = static_cast<double>(s.m), t = static_cast<double>(tau), L = s.lambda_max;
    const double rt = std::pow(rho, t);
    GammaBounds g;
    g.b1 = 1.0 / psi(static_cast<double>(s.mu), L, tau, rho, s.m);
    g.b2 = m * (rho - 1.0) / (2.0 * L * rt * rho);
    g.b3 = m * std::sqrt((rho - 1.0) / (rt * (m * s.alpha * s.alpha + L * L * t * rt)));
    g.gamma = std::min({g.b1, g.b2, g.b3});
    return g;
}

StepParams corollary_params(const SystemStats& s, index_t tau) {
    need_core(s);
    if (tau < 0) fail(ErrorCode::InvalidArgument, "tau must be >= 0");
    const double m = static_cast<double>(s.m);
    const double lhs = 2.0 * std::numbers::e * s.lambda_max * static_cast<double>(tau + 1) / m;
    StepParams p;
    p.tau = tau;
    p.feasible = lhs <= 1.0;
    p.rho = 1.0 + lhs;
    p.psi = psi(static_cast<double>(s.mu), s.lambda_max, tau, p.rho, s.m);
    if (p.feasible) {
        p.gamma_bounds = gamma_bounds(s, tau, p.rho);
        p.gamma = 1.0 / p.psi;
        if (s.lambda_min) {
            if (!(p.gamma < 2.0 / p.psi)) fail(ErrorCode::StepTooLarge, "gamma must stay below 2/psi");
            p.rate_iter = 1.0 - *s.lambda_min * p.gamma * (2.0 - p.gamma * p.psi) / m;
            p.rate_simplified = 1.0 - *s.lambda_min / (m * (static_cast<double>(s.mu) + 1.0));
        }
    }
    return p;
}

index_t max_feasible_tau(index_t m, double lambda_max) {
    return static_cast<index_t>(std::floor(static_cast<double>(m) / (2.0 * std::numbers::e * lambda_max))) - 1;
}

}  // namespace asyrk
